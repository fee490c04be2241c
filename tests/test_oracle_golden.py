"""The CPU oracle (oracle/laze_port.py) against vectors produced by the REAL reference
(tests/golden/make_golden.py: laze eager context + lazy compile pipeline), and against the
reference's own known-answer tests for the array ops on this path.  Runs everywhere (no GPU, no
/root/reference needed)."""
import glob
import os

import numpy as np
import pytest

from oracle.laze_port import NumpyArrayContext, OutOfBoundsIndex, checked_take, rel_err
from paper_2512_17101_b200.operators import EulerOperator, NavierStokesOperator, rk4_step
from tests.common import FARFIELD, make_dcoll
from tests.common import GOLDEN_CASES as CASES

GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_operator_program_matches_reference(case):
    name, dim, order, n, bc, opname, kw, _ = case
    g = np.load(os.path.join(GOLD, name + ".npz"))
    actx = NumpyArrayContext()
    d = make_dcoll(actx, dim, order, n, bc)
    # connectivity / index maps: bit-exact
    assert np.array_equal(d.vmap_m_host, g["vmap_m"]) and np.array_equal(d.vmap_p_host, g["vmap_p"])
    assert np.array_equal(d.bc_kind_host, g["bc_kind"])
    op = (EulerOperator if opname == "euler" else NavierStokesOperator)(d, farfield=FARFIELD[dim], **kw)
    rhs = d.to_numpy(op.rhs(d.from_numpy(g["q0"])))
    assert np.array_equal(rhs, g["eager_rhs"])                  # same NumPy calls as the eager reference
    assert rel_err(rhs, g["lazy_rhs"]) <= 1e-12                 # the reference's own pipeline-vs-oracle bar
    if opname == "ns":
        grad = d.to_numpy(op.grad(d.from_numpy(g["q0"])))
        assert np.array_equal(grad, g["eager_grad"])
        assert rel_err(grad, g["lazy_grad"]) <= 1e-12
        # both arrangements of the scheme (operators.py) against the reference's eager and lazy results
        alt = d.to_numpy(op.rhs_grad_form(d.from_numpy(g["q0"])))
        assert np.array_equal(alt, g["eager_rhs_grad_form"])
        assert rel_err(alt, g["lazy_rhs_grad_form"]) <= 1e-12
        assert rel_err(alt, rhs) <= 1e-13
        T = np.asarray(op.flux(d.from_numpy(g["q0"])))
        assert np.array_equal(T, g["eager_flux"]) and rel_err(T, g["lazy_flux"]) <= 1e-12


def test_rk4_matches_reference():
    g = np.load(os.path.join(GOLD, "euler2d_p3_rk4_20steps.npz"))
    actx = NumpyArrayContext()
    d = make_dcoll(actx, 2, 3, 4, "periodic")
    op = EulerOperator(d)
    q, t, dt = d.from_numpy(g["q0"]), 0.0, float(g["dt"])
    for _ in range(20):
        q = rk4_step(op.rhs, q, t, dt)
        t += dt
    assert np.array_equal(d.to_numpy(q), g["q"])


def test_reference_known_answers():
    g = np.load(os.path.join(GOLD, "array_ops.npz"))
    actx = NumpyArrayContext()
    # gather v=[10..14], sel=[4,0,2]   (/root/reference/pkg/tests/test_scalar_ir.py:160-170)
    v = actx.from_numpy(np.array([10.0, 11.0, 12.0, 13.0, 14.0]))
    sel = actx.from_numpy(np.array([4, 0, 2], dtype=np.int64))
    assert np.array_equal(v[sel], [14.0, 10.0, 12.0]) and np.array_equal(v[sel], g["gather"])
    # einsum -> reshape -> slice        (/root/reference/pkg/tests/test_frontend.py:126-134)
    comp = actx.np.einsum("ij,jk->ik", g["a"], g["b"]).reshape(5, 3)[1:4]
    assert rel_err(comp, g["einsum_reshape_slice"]) <= 1e-15
    # out-of-range gather raises         (/root/reference/pkg/tests/test_backend.py:72-80)
    with pytest.raises(OutOfBoundsIndex):
        checked_take(np.arange(5.0), np.array([0, 5]))
    # Fig.-7 flux fold: 2*(3/6)*(1+3) == 4 (/root/reference/pkg/tests/test_graph_passes.py:75-90)
    assert actx.np.multiply(actx.np.multiply(2.0, actx.np.divide(3.0, 6.0)), actx.np.add(1.0, 3.0)) == 4.0


def test_golden_files_present():
    assert len(glob.glob(os.path.join(GOLD, "*.npz"))) >= 7
