"""Reference-independent checks of the DG physics (the reference pins array-op semantics only;
SURVEY.md §7 hard part 2): exactness of the reference matrices, free-stream preservation,
conservation, convergence of the isentropic vortex at order p+1."""
import itertools

import numpy as np
import pytest

from oracle.laze_port import NumpyArrayContext
from paper_2512_17101_b200.dg.simplex import simplex_element
from paper_2512_17101_b200.operators import EulerOperator, NavierStokesOperator, rk4_step
from tests.common import make_dcoll


@pytest.mark.parametrize("dim,p", [(2, 1), (2, 3), (2, 4), (3, 1), (3, 2), (3, 3), (3, 4)])
def test_reference_matrices(dim, p):
    el = simplex_element(dim, p)
    r = el.rst
    for e in itertools.product(range(p + 1), repeat=dim):
        if sum(e) > p:
            continue
        f = np.prod([r[k] ** e[k] for k in range(dim)], axis=0)
        for k in range(dim):
            ee = list(e)
            if ee[k] == 0:
                df = np.zeros_like(f)
            else:
                ee[k] -= 1
                df = e[k] * np.prod([r[m] ** ee[m] for m in range(dim)], axis=0)
            assert np.abs(el.D[k] @ f - df).max() < 1e-12
    vol = {2: 2.0, 3: 4.0 / 3.0}[dim]
    assert abs(el.mass.sum() - vol) < 1e-13
    assert np.abs(el.mass @ el.Sw[0] - el.D[0].T @ el.mass).max() < 1e-13
    # integration by parts on the reference element: M D_r + D_r^T M = sum_f nhat_{r,f} E_f
    # checked through lift: 1^T M lift(e) = face integral
    one = np.ones(el.Np)
    for f in range(el.Nf):
        face_int = one @ el.mass @ el.lift[:, f * el.Nfp:(f + 1) * el.Nfp]
        assert abs(face_int.sum() - {2: 2.0, 3: 2.0}[dim]) < 1e-12      # area of the standard face
    # face-node permutation tables are permutations, identity first
    assert np.array_equal(el.face_perms[0], np.arange(el.Nfp))
    for row in el.face_perms:
        assert sorted(row.tolist()) == list(range(el.Nfp))


@pytest.mark.parametrize("dim,bc", [(2, "periodic"), (3, "periodic"), (3, "farfield")])
def test_free_stream_preservation(dim, bc):
    actx = NumpyArrayContext()
    d = make_dcoll(actx, dim, 3, 3, bc)
    qf = np.array([1.2, 2.9, 0.3, -0.2, 0.1][:dim + 2])
    q = d.from_numpy(np.broadcast_to(qf[:, None, None], (dim + 2, d.nelements, d.Np)))
    for Op in (EulerOperator, NavierStokesOperator):
        op = Op(d, farfield=qf)
        assert np.abs(d.to_numpy(op.rhs(q))).max() < 5e-12


def test_conservation_periodic():
    """sum_e J_e 1^T M rhs_e == 0 for every conserved field on a periodic mesh."""
    actx = NumpyArrayContext()
    d = make_dcoll(actx, 3, 3, 3, "periodic")
    from tests.common import smooth_state
    q = d.from_numpy(smooth_state(d.nodes()))
    for Op, kw in [(EulerOperator, {}), (NavierStokesOperator, {"mu": 2e-2})]:
        r = d.to_numpy(Op(d, **kw).rhs(q))
        total = np.einsum("i,ij,cej,e->c", np.ones(d.Np), d.element.mass, r, d.geo.jac)
        assert np.abs(total).max() < 1e-11


def _vortex(x, t, gamma=1.4, beta=5.0):
    xr, yr = x[0] - 5.0 - t, x[1]
    r2 = xr ** 2 + yr ** 2
    ex = np.exp(1 - r2)
    u = 1.0 - beta * ex * yr / (2 * np.pi)
    v = beta * ex * xr / (2 * np.pi)
    rho = (1 - (gamma - 1) / (16 * gamma * np.pi ** 2) * beta ** 2 * np.exp(2 * (1 - r2))) ** (1 / (gamma - 1))
    p = rho ** gamma
    return np.stack([rho, p / (gamma - 1) + 0.5 * rho * (u * u + v * v), rho * u, rho * v])


def test_isentropic_vortex_convergence():
    """BASELINE configs[0]: 2D Euler isentropic vortex, order 3, RK4; error falls at ~h^(p+1)."""
    from paper_2512_17101_b200 import DGDiscretization, box_mesh
    actx = NumpyArrayContext()
    errs = []
    for n in (8, 16):
        mesh = box_mesh((n, n), (0.0, -5.0), (10.0, 5.0), periodic=(True, True))
        d = DGDiscretization(actx, mesh, 3)
        op = EulerOperator(d)
        q = d.interp(lambda x: _vortex(x, 0.0))
        T = 0.2
        nst = int(np.ceil(T / (0.02 * 8 / n)))
        dt, t = T / nst, 0.0
        for _ in range(nst):
            q = rk4_step(op.rhs, q, t, dt)
            t += dt
        errs.append(d.norm_l2(d.to_numpy(q) - _vortex(d.nodes(), T)))
    rate = np.log2(errs[0] / errs[1])
    assert rate > 2.5, (errs, rate)


@pytest.mark.parametrize("dims,per", [((4, 4, 4), True), ((5, 4, 3), False), ((6, 5), True)])
def test_mesh_connectivity_with_two_level_face_keys(dims, per, monkeypatch):
    """Meshes whose packed face keys (nvert**dim) would overflow 62 bits (periodic 3D boxes beyond n = 118) rank the
    partial keys first; forced here on small meshes, the connectivity must not change."""
    from paper_2512_17101_b200.dg import mesh as M
    dim = len(dims)
    a = M.box_mesh(dims, (-1,) * dim, (1,) * dim, periodic=(per,) * dim)
    monkeypatch.setattr(M, "_KEY_LIMIT", 2.0 ** 9)
    b = M.box_mesh(dims, (-1,) * dim, (1,) * dim, periodic=(per,) * dim)
    for f in ("nbr_elem", "nbr_face", "nbr_perm", "btag"):
        assert np.array_equal(getattr(a, f), getattr(b, f)), f
