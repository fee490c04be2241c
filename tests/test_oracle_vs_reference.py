"""Pins the oracle port against the REAL reference package when it is mounted (build container);
skipped on the GPU box, where /root/reference does not exist."""
import os
import sys

import numpy as np
import pytest

REF = "/root/reference/pkg/src"
pytestmark = pytest.mark.skipif(not os.path.isdir(REF), reason="reference not mounted")


@pytest.fixture(scope="module")
def laze():
    sys.path.insert(0, REF)
    import laze as mod
    return mod


def _run(actx, dim, order, n, bc, Op, kw, q0):
    from tests.common import FARFIELD, make_dcoll
    d = make_dcoll(actx, dim, order, n, bc)
    op = Op(d, farfield=FARFIELD[dim], **kw)
    return np.asarray(actx.to_numpy(op.rhs(d.from_numpy(q0)).data))


@pytest.mark.parametrize("dim,order,n,bc", [(2, 3, 3, "mixed"), (3, 2, 2, "mixed"), (3, 3, 3, "periodic")])
def test_port_equals_reference_eager(laze, dim, order, n, bc):
    from oracle.laze_port import NumpyArrayContext
    from paper_2512_17101_b200.operators import EulerOperator, NavierStokesOperator
    from tests.common import make_dcoll, random_state
    probe = make_dcoll(NumpyArrayContext(), dim, order, n, bc)
    q0 = random_state(dim, probe.nelements, probe.Np, seed=3)
    for Op, kw in [(EulerOperator, {}), (NavierStokesOperator, {"mu": 2e-2})]:
        a = _run(NumpyArrayContext(), dim, order, n, bc, Op, kw, q0)
        b = _run(laze.ArrayContext(mode="eager"), dim, order, n, bc, Op, kw, q0)
        assert np.array_equal(a, b)


def test_program_is_legal_under_lazy_tracing(laze):
    """The operator program obeys the reference's tracing rules (<=1 index array per subscript,
    gather depth <= 1, rank <= 8) and its compiled pipeline agrees with the port to 1e-12."""
    from oracle.laze_port import NumpyArrayContext, rel_err
    from paper_2512_17101_b200.operators import NavierStokesOperator
    from tests.common import make_dcoll, random_state
    probe = make_dcoll(NumpyArrayContext(), 2, 2, 3, "mixed")
    q0 = random_state(2, probe.nelements, probe.Np, seed=4)
    a = _run(NumpyArrayContext(), 2, 2, 3, "mixed", NavierStokesOperator, {"mu": 2e-2}, q0)
    b = _run(laze.ArrayContext(mode="lazy"), 2, 2, 3, "mixed", NavierStokesOperator, {"mu": 2e-2}, q0)
    assert rel_err(b, a) <= 1e-12


def test_outlined_functions_become_call_nodes(laze):
    """`actx.outline` turns each DG function into a Call to a FunctionDefinition named like the
    C-ABI kernel that replaces it (the plugin boundary)."""
    from laze.adfg import CallResult
    from paper_2512_17101_b200.operators import NavierStokesOperator
    from tests.common import make_dcoll, random_state
    actx = laze.ArrayContext(mode="lazy")
    d = make_dcoll(actx, 2, 1, 3, "periodic")
    op = NavierStokesOperator(d, mu=1e-2)
    q = d.from_numpy(random_state(2, d.nelements, d.Np))
    g = op.grad(q)
    assert isinstance(g.data.node, CallResult) and g.data.node.call.function.name == "dg_ns_grad"
    r = op.rhs(q)
    assert r.data.node.call.function.name == "dg_ns_div"
    T = op.flux(q)
    assert isinstance(T.node, CallResult) and T.node.call.function.name == "dg_ns_flux"
    r = op.rhs_grad_form(q)
    assert r.data.node.call.function.name == "dg_ns_rhs"
