"""GPU parity: the operator program on B200ArrayContext (fused sm_100a kernels through the C ABI)
against the CPU oracle (oracle/laze_port.py) on identical meshes and states.

Tolerances are the north star's: max relative error <= 1e-12 per RHS evaluation and <= 1e-10 after
100 RK4 steps, in the reference's norm max|d| / max(max|ref|, 1)
(/root/reference/pkg/tests/test_acceptance.py:38-41); index maps bit-exact.
"""
import numpy as np
import pytest

from oracle.laze_port import NumpyArrayContext, rel_err
from paper_2512_17101_b200.operators import EulerOperator, NavierStokesOperator, rk4_step
from tests.common import FARFIELD, make_dcoll, random_state, smooth_state

pytestmark = pytest.mark.gpu
TOL_RHS = 1e-12
TOL_RK = 1e-10


@pytest.fixture(scope="module")
def gpu():
    from paper_2512_17101_b200 import B200ArrayContext
    return B200ArrayContext()


CASES = [
    (3, 3, 3, "periodic"), (3, 3, 2, "mixed"), (3, 3, 3, "farfield"),
    (3, 4, 3, "periodic"), (3, 2, 3, "mixed"), (3, 1, 3, "periodic"), (3, 4, 2, "mixed"),
    (2, 3, 4, "periodic"), (2, 3, 4, "mixed"), (2, 1, 3, "farfield"), (2, 2, 5, "periodic"), (2, 4, 3, "mixed"),
]


def _both(dim, order, n, bc):
    cpu = NumpyArrayContext()
    return make_dcoll(cpu, dim, order, n, bc), None


@pytest.mark.parametrize("dim,order,n,bc", CASES)
def test_index_maps_bit_exact(gpu, dim, order, n, bc):
    """Compressed device connectivity expands to exactly the host int64 maps."""
    import ctypes as C
    from paper_2512_17101_b200 import _cabi
    from paper_2512_17101_b200.fused import get_disc
    d = make_dcoll(gpu, dim, order, n, bc)
    q = d.from_numpy(random_state(dim, d.nelements, d.Np)).data
    disc = get_disc(gpu, dim, q, 0, d.Sw, d.drdx, d.lift, d.normals, d.fscale, d.vmap_m, d.vmap_p, d.bc_kind)
    vm = gpu.empty(d.vmap_m.shape, 1)
    vp = gpu.empty(d.vmap_p.shape, 1)
    _cabi.check(gpu.lib.dgb_disc_expand_maps(disc.handle, vm.ptr, vp.ptr, gpu._st))
    assert np.array_equal(gpu.to_numpy(vm), d.vmap_m_host.reshape(-1))
    assert np.array_equal(gpu.to_numpy(vp), d.vmap_p_host.reshape(-1))


@pytest.mark.parametrize("dim,order,n,bc", CASES)
def test_rhs_parity(gpu, dim, order, n, bc):
    cpu = NumpyArrayContext()
    dc, dg = make_dcoll(cpu, dim, order, n, bc), make_dcoll(gpu, dim, order, n, bc)
    for seed, q0 in [(1, random_state(dim, dc.nelements, dc.Np, seed=1)), (0, smooth_state(dc.nodes()))]:
        for Op, kw in [(EulerOperator, {}), (NavierStokesOperator, {"mu": 2e-2})]:
            oc = Op(dc, farfield=FARFIELD[dim], **kw)
            og = Op(dg, farfield=FARFIELD[dim], **kw)
            ref = dc.to_numpy(oc.rhs(dc.from_numpy(q0)))
            got = dg.to_numpy(og.rhs(dg.from_numpy(q0)))
            assert got.shape == ref.shape
            assert rel_err(got, ref) <= TOL_RHS, (Op.__name__, seed, rel_err(got, ref))
            if Op is NavierStokesOperator:
                gref = dc.to_numpy(oc.grad(dc.from_numpy(q0)))
                ggot = dg.to_numpy(og.grad(dg.from_numpy(q0)))
                assert rel_err(ggot, gref) <= TOL_RHS, ("grad", seed, rel_err(ggot, gref))
                # pass 1 of the flux arrangement on its own, and the gradient arrangement end to end
                tref = np.asarray(cpu.to_numpy(oc.flux(dc.from_numpy(q0))))
                tgot = np.asarray(gpu.to_numpy(og.flux(dg.from_numpy(q0))))
                assert rel_err(tgot, tref) <= TOL_RHS, ("flux planes", seed, rel_err(tgot, tref))
                got2 = dg.to_numpy(og.rhs_grad_form(dg.from_numpy(q0)))
                assert rel_err(got2, ref) <= TOL_RHS, ("grad form", seed, rel_err(got2, ref))


@pytest.mark.parametrize("dim,order,n,bc", [(3, 3, 2, "mixed"), (2, 3, 3, "mixed"), (3, 2, 3, "periodic")])
def test_generic_ops_parity(gpu, dim, order, n, bc):
    """The same program with fused dispatch switched off runs op by op on the generic device
    kernels (einsum, gather, where, stack, reshape, elementwise) and must agree as well."""
    from paper_2512_17101_b200 import B200ArrayContext
    plain = B200ArrayContext()
    plain._fused = {}
    cpu = NumpyArrayContext()
    dc, dg = make_dcoll(cpu, dim, order, n, bc), make_dcoll(plain, dim, order, n, bc)
    q0 = random_state(dim, dc.nelements, dc.Np, seed=3)
    for Op, kw in [(EulerOperator, {}), (NavierStokesOperator, {"mu": 2e-2})]:
        ref = dc.to_numpy(Op(dc, farfield=FARFIELD[dim], **kw).rhs(dc.from_numpy(q0)))
        got = dg.to_numpy(Op(dg, farfield=FARFIELD[dim], **kw).rhs(dg.from_numpy(q0)))
        assert rel_err(got, ref) <= TOL_RHS, (Op.__name__, rel_err(got, ref))


@pytest.mark.parametrize("dim,order,n,Op,kw", [
    (2, 3, 4, EulerOperator, {}), (3, 3, 3, EulerOperator, {}), (3, 3, 3, NavierStokesOperator, {"mu": 1e-2})])
def test_rk4_100_steps(gpu, dim, order, n, Op, kw):
    cpu = NumpyArrayContext()
    dc, dg = make_dcoll(cpu, dim, order, n, "periodic"), make_dcoll(gpu, dim, order, n, "periodic")
    q0 = smooth_state(dc.nodes())
    oc, og = Op(dc, **kw), Op(dg, **kw)
    qc, qg = dc.from_numpy(q0), dg.from_numpy(q0)
    dt = 2e-3
    t = 0.0
    for _ in range(100):
        qc = rk4_step(oc.rhs, qc, t, dt)
        qg = rk4_step(og.rhs, qg, t, dt)
        t += dt
    ref, got = dc.to_numpy(qc), dg.to_numpy(qg)
    assert np.all(np.isfinite(got))
    assert rel_err(got, ref) <= TOL_RK, rel_err(got, ref)


def test_tail_block_and_odd_sizes(gpu):
    """Element counts that are not multiples of the CTA block (ragged last block)."""
    cpu = NumpyArrayContext()
    for n in (1, 2):   # E = 6, 48 in 3D (non-periodic so tiny meshes are legal)
        dc, dg = make_dcoll(cpu, 3, 3, n, "farfield"), make_dcoll(gpu, 3, 3, n, "farfield")
        q0 = random_state(3, dc.nelements, dc.Np, seed=7)
        ref = dc.to_numpy(NavierStokesOperator(dc, farfield=FARFIELD[3], mu=1e-2).rhs(dc.from_numpy(q0)))
        got = dg.to_numpy(NavierStokesOperator(dg, farfield=FARFIELD[3], mu=1e-2).rhs(dg.from_numpy(q0)))
        assert rel_err(got, ref) <= TOL_RHS


def test_out_of_bounds_map_rejected(gpu):
    """An index map leaving [0, E*Np) raises OutOfBoundsIndex at upload, like the reference's
    bounds-checked gather (/root/reference/pkg/tests/test_backend.py:72-80)."""
    from paper_2512_17101_b200 import errors
    d = make_dcoll(gpu, 3, 2, 2, "farfield")
    bad = d.vmap_p_host.reshape(-1).copy()
    bad[5] = d.nelements * d.Np + 3
    d.vmap_p = gpu.from_numpy(bad)
    op = EulerOperator(d, farfield=FARFIELD[3])
    with pytest.raises(errors.OutOfBoundsIndex):
        op.rhs(d.from_numpy(random_state(3, d.nelements, d.Np)))
    bad2 = d.vmap_p_host.reshape(-1).copy()
    bad2[[0, 1]] = bad2[[1, 0]]
    d.vmap_p = gpu.from_numpy(bad2)
    with pytest.raises(errors.BindingMismatch):
        EulerOperator(d, farfield=FARFIELD[3]).rhs(d.from_numpy(random_state(3, d.nelements, d.Np)))


@pytest.mark.timeout(900)
@pytest.mark.parametrize("order,n,bc", [(3, 16, "periodic"), (3, 24, "mixed"), (4, 16, "mixed")])
def test_midsize_parity(gpu, order, n, bc):
    """Direct oracle comparison at sizes where the persistent-kernel machinery is exercised: 24.6 k /
    82.9 k elements = 5-23 blocks per warp of a full grid (work tickets two deep, double-buffered
    staging across blocks, early gathers of the next block), mixed boundaries, and the odd-Np order-4
    path.  Same 1e-12 bar as the small cases."""
    cpu = NumpyArrayContext()
    dc, dg = make_dcoll(cpu, 3, order, n, bc), make_dcoll(gpu, 3, order, n, bc)
    q0 = random_state(3, dc.nelements, dc.Np, seed=11)
    q0s = smooth_state(dc.nodes())
    for Op, kw, qq in [(NavierStokesOperator, {"mu": 2e-2}, q0), (EulerOperator, {}, q0),
                       (NavierStokesOperator, {"mu": 1e-3}, q0s)]:
        oc = Op(dc, farfield=FARFIELD[3], **kw)
        og = Op(dg, farfield=FARFIELD[3], **kw)
        ref = dc.to_numpy(oc.rhs(dc.from_numpy(qq)))
        got = dg.to_numpy(og.rhs(dg.from_numpy(qq)))
        assert rel_err(got, ref) <= TOL_RHS, (Op.__name__, rel_err(got, ref))
        if Op is NavierStokesOperator and qq is q0:
            tref = np.asarray(cpu.to_numpy(oc.flux(dc.from_numpy(qq))))
            tgot = np.asarray(gpu.to_numpy(og.flux(dg.from_numpy(qq))))
            assert rel_err(tgot, tref) <= TOL_RHS, ("flux planes", rel_err(tgot, tref))
            # RK-fused epilogue at this size: out1 = a1*x1 + b1*rhs, out2 = a2*x2 + b2*rhs
            qd = dg.from_numpy(qq)
            o1, o2 = og.rhs_rk(qd, qd, qd, (1.0, 0.25, 0.5, -2.0))
            assert rel_err(dg.to_numpy(o1), qq + 0.25 * ref) <= TOL_RHS
            assert rel_err(dg.to_numpy(o2), 0.5 * qq - 2.0 * ref) <= TOL_RHS


@pytest.mark.parametrize("dim,order,n,bc", [(3, 3, 2, "mixed"), (3, 3, 12, "mixed"), (3, 4, 6, "mixed"), (3, 2, 5, "periodic"),
                                            (3, 1, 5, "mixed"), (2, 3, 9, "mixed"), (2, 4, 7, "periodic"), (2, 1, 7, "farfield")])
def test_tma_staged_pass2_is_bitwise_equal_to_cp_async_pass2(gpu, dim, order, n, bc, monkeypatch):
    """k_nsdiv8 (default: rows by TMA boxes, neighbours through the 32-bit gather map, all rounds of a block in
    flight) against k_nsdiv3 (cp.async staging, connectivity decoded per node): same arithmetic in the same order,
    so the right-hand sides and the fused RK outputs must be bitwise equal -- odd Np (shifted boxes) included."""
    d = make_dcoll(gpu, dim, order, n, bc)
    op = NavierStokesOperator(d, farfield=FARFIELD[dim], mu=2e-2)
    q = d.from_numpy(random_state(dim, d.nelements, d.Np, seed=3))
    outs = {}
    for k in ("3", "8"):
        monkeypatch.setenv("DGB_DIV_KERNEL", k)
        o1, o2 = op.rhs_rk(q, q, q, (1.0, 0.25, 0.5, -2.0))
        outs[k] = (d.to_numpy(op.rhs(q)), d.to_numpy(o1), d.to_numpy(o2))
    for a, b in zip(outs["3"], outs["8"]):
        assert np.isfinite(a).all() and np.array_equal(a, b)


def test_run_to_run_bitwise(gpu):
    """No atomics anywhere on the path: two evaluations are bitwise identical."""
    d = make_dcoll(gpu, 3, 3, 3, "periodic")
    op = NavierStokesOperator(d, mu=1e-2)
    q = d.from_numpy(random_state(3, d.nelements, d.Np))
    a = d.to_numpy(op.rhs(q))
    b = d.to_numpy(op.rhs(q))
    assert np.array_equal(a, b)


def test_gpu_matches_reference_golden(gpu):
    """GPU results against vectors produced by the REAL reference package (tests/golden/)."""
    import os
    from tests.common import GOLDEN_CASES as GOLDEN
    gold = os.path.join(os.path.dirname(__file__), "golden")
    for name, dim, order, n, bc, opname, kw, _ in GOLDEN:
        g = np.load(os.path.join(gold, name + ".npz"))
        d = make_dcoll(gpu, dim, order, n, bc)
        op = (EulerOperator if opname == "euler" else NavierStokesOperator)(d, farfield=FARFIELD[dim], **kw)
        got = d.to_numpy(op.rhs(d.from_numpy(g["q0"])))
        assert rel_err(got, g["eager_rhs"]) <= TOL_RHS, name
        assert rel_err(got, g["lazy_rhs"]) <= TOL_RHS, name
        if opname == "ns":
            assert rel_err(d.to_numpy(op.grad(d.from_numpy(g["q0"]))), g["eager_grad"]) <= TOL_RHS, name
            assert rel_err(d.to_numpy(op.rhs_grad_form(d.from_numpy(g["q0"]))), g["eager_rhs_grad_form"]) <= TOL_RHS, name
            assert rel_err(gpu.to_numpy(op.flux(d.from_numpy(g["q0"]))), g["eager_flux"]) <= TOL_RHS, name


@pytest.mark.parametrize("dim,order,n,Op,kw", [(3, 3, 3, EulerOperator, {}), (3, 3, 3, NavierStokesOperator, {"mu": 1e-2}),
                                                (2, 4, 3, NavierStokesOperator, {"mu": 1e-2})])
def test_fused_rk_stage(gpu, dim, order, n, Op, kw):
    """RK stage update fused into the RHS epilogue (dgb_*_rhs_rk) == the same program on the oracle,
    and == the unfused classical RK4 to round-off."""
    from paper_2512_17101_b200 import rk4_step_fused
    cpu = NumpyArrayContext()
    dc, dg = make_dcoll(cpu, dim, order, n, "periodic"), make_dcoll(gpu, dim, order, n, "periodic")
    q0 = smooth_state(dc.nodes())
    oc, og = Op(dc, **kw), Op(dg, **kw)
    qc, qg, qu = dc.from_numpy(q0), dg.from_numpy(q0), dg.from_numpy(q0)
    t, dt = 0.0, 2e-3
    for _ in range(10):
        qc = rk4_step_fused(oc, qc, t, dt)
        qg = rk4_step_fused(og, qg, t, dt)
        qu = rk4_step(og.rhs, qu, t, dt)
        t += dt
    assert rel_err(dg.to_numpy(qg), dc.to_numpy(qc)) <= 1e-12
    assert rel_err(dg.to_numpy(qg), dg.to_numpy(qu)) <= 1e-12
    if Op is NavierStokesOperator:       # the gradient arrangement's fused stage update
        c = (1.0, 0.5 * dt, 1.0, dt / 6.0)
        a1, a2 = og.rhs_rk(qg, qg, qu, c)
        b1, b2 = og.rhs_rk_grad_form(qg, qg, qu, c)
        assert rel_err(dg.to_numpy(b1), dg.to_numpy(a1)) <= 1e-12
        assert rel_err(dg.to_numpy(b2), dg.to_numpy(a2)) <= 1e-12


@pytest.mark.parametrize("dim,order,n,per,nparts", [(3, 3, 3, True, 2), (2, 3, 4, False, 3), (3, 3, 4, True, 4), (3, 3, 4, False, 8),
                                                         (3, 4, 3, True, 2), (3, 4, 4, False, 4), (3, 4, 4, True, 8)])
def test_ghost_elements_on_device(gpu, dim, order, n, per, nparts):
    """Partitioned meshes on the device: halo packing kernel + ghost-element gathers in the fused
    kernels, with the exchange itself looped back on the host (this box has one GPU)."""
    from paper_2512_17101_b200 import DGDiscretization, box_mesh
    from paper_2512_17101_b200.dg.partition import partition_elements, rank_mesh
    from paper_2512_17101_b200.discretization import BC_FARFIELD, BC_WALL
    from paper_2512_17101_b200.halo import HaloExchange
    cpu = NumpyArrayContext()
    mesh = box_mesh((n,) * dim, (-1,) * dim, (1,) * dim, periodic=(per,) * dim)
    bc = None if per else {k: (BC_WALL if k % 2 else BC_FARFIELD) for k in range(1, 2 * dim + 1)}
    d = DGDiscretization(cpu, mesh, order, bc_map=bc)
    q0 = random_state(dim, d.nelements, d.Np, seed=5)
    ref = d.to_numpy(NavierStokesOperator(d, farfield=FARFIELD[dim], mu=2e-2).rhs(d.from_numpy(q0)))
    part = partition_elements(mesh, nparts)
    locs = [rank_mesh(mesh, part, r) for r in range(nparts)]
    ds = [DGDiscretization(gpu, m, order, bc_map=bc, ghost_elements=p.nghost) for m, p in locs]
    ops = [NavierStokesOperator(dd, farfield=FARFIELD[dim], mu=2e-2) for dd in ds]
    qs = [ds[r].from_numpy(q0[:, p.global_ids, :]) for r, (_, p) in enumerate(locs)]
    halos = [HaloExchange(gpu, p, object(), d.Np) for _, p in locs]

    def exchange(fields):
        packed = {}
        for r, (_, p) in enumerate(locs):
            for k, peer in enumerate(p.peers):
                packed[(r, peer)] = gpu.to_numpy(halos[r]._pack(fields[r], k))     # device pack kernel
        out = []
        for r, (_, p) in enumerate(locs):
            g = np.empty(tuple(fields[r].shape[:-2]) + (p.nghost, d.Np))
            for k, peer in enumerate(p.peers):
                a, b = p.recv_slots[k]
                g[..., a:b, :] = packed[(peer, r)]
            out.append(gpu.from_numpy(g))
        return out

    gh = exchange([q.data for q in qs])
    gqs = [ops[r].grad(qs[r], gh[r]) for r in range(nparts)]
    ggh = exchange([g.data for g in gqs])
    Ts = [ops[r].flux(qs[r], gh[r]) for r in range(nparts)]
    tgh = exchange(Ts)
    for form in ("flux", "grad"):
        full = np.empty_like(ref)
        for r, (_, p) in enumerate(locs):
            if form == "flux":
                out = ops[r].rhs(qs[r], ghost=gh[r], halo_fn=lambda T, r=r: tgh[r])
            else:
                out = ops[r].rhs_grad_form(qs[r], ghost=gh[r], halo_fn=lambda gq, r=r: ggh[r])
            full[:, p.global_ids, :] = ds[r].to_numpy(out)
        assert rel_err(full, ref) <= TOL_RHS, form


@pytest.mark.timeout(900)
def test_full_size_properties(gpu):
    """BASELINE configs[2] at full size (3D NS p3, 94^3 Kuhn box, 99.67M DOFs), where the oracle cannot run:
    size-independent properties instead -- free-stream preservation, discrete conservation on the
    periodic mesh, agreement of the two arrangements of the scheme (independent kernels), linearity
    of the RK-fused epilogue, and run-to-run bitwise reproducibility."""
    from tests.common import smooth_state
    d = make_dcoll(gpu, 3, 3, 94, "periodic")
    E, Np = d.nelements, d.Np
    assert E * Np == 99670080
    op = NavierStokesOperator(d, mu=1e-3)
    # free stream: a constant state has zero right-hand side
    qf = np.array([1.2, 2.9, 0.3, -0.2, 0.1])
    qc = d.from_numpy(np.broadcast_to(qf[:, None, None], (5, E, Np)))
    assert d.norm_inf(op.rhs(qc)) < 5e-11
    del qc
    # smooth state: conservation, arrangement agreement, reproducibility
    q = d.from_numpy(smooth_state(d.nodes()))
    r = op.rhs(q)
    rh = d.to_numpy(r)
    assert np.all(np.isfinite(rh))
    w = np.einsum("i,ij->j", np.ones(Np), d.element.mass)
    total = np.einsum("cej,j,e->c", rh, w, d.geo.jac)
    scale = np.einsum("cej,j,e->c", np.abs(rh), w, d.geo.jac)
    assert np.all(np.abs(total) <= 1e-12 * np.maximum(scale, 1.0)), (total, scale)
    # Two independent kernel pairs, no oracle.  The 1e-12 per-RHS tolerance is checked against the oracle
    # on the parity meshes (n <= 5 above); round-off of a derivative operator grows like 1/h, and h here
    # is 30x smaller, so the bar between two algebraically equal arrangements is scaled accordingly.
    r2 = d.to_numpy(op.rhs_grad_form(q))
    assert rel_err(r2, rh) <= TOL_RHS * 94 / 3
    del r2
    assert np.array_equal(d.to_numpy(op.rhs(q)), rh)
    # fused stage update == a*x + b*rhs
    o1, o2 = op.rhs_rk(q, q, r, (1.0, 0.25, 0.5, -2.0))
    assert rel_err(d.to_numpy(o1), smooth_state(d.nodes()) + 0.25 * rh) <= 1e-13
    assert rel_err(d.to_numpy(o2), 0.5 * rh - 2.0 * rh) <= 1e-13


@pytest.mark.parametrize("Op,kw,dim,order,n", [(NavierStokesOperator, {"mu": 1e-2}, 3, 3, 3), (EulerOperator, {}, 3, 3, 3),
                                                (NavierStokesOperator, {"mu": 1e-2}, 2, 4, 3)])
def test_device_rk4_driver(gpu, Op, kw, dim, order, n):
    """DeviceRK4 (all stage storage owned, C ABI called directly, whole step captured in one CUDA
    graph) == classical RK4 of the same operator program on the oracle, and graph replay == eager launches."""
    from paper_2512_17101_b200 import DeviceRK4
    cpu = NumpyArrayContext()
    dc, dg = make_dcoll(cpu, dim, order, n, "periodic"), make_dcoll(gpu, dim, order, n, "periodic")
    q0 = smooth_state(dc.nodes())
    oc, og = Op(dc, **kw), Op(dg, **kw)
    dt, nsteps = 2e-3, 25
    qc, t = dc.from_numpy(q0), 0.0
    for _ in range(nsteps):
        qc = rk4_step(oc.rhs, qc, t, dt)
        t += dt
    ref = dc.to_numpy(qc)
    launches0 = gpu.launch_count
    graph = DeviceRK4(og, dg.from_numpy(q0), dt, use_graph=True).step(nsteps)
    eager = DeviceRK4(og, dg.from_numpy(q0), dt, use_graph=False).step(nsteps)
    got_g, got_e = dg.to_numpy(graph.state), dg.to_numpy(eager.state)
    assert graph.graph is not None and abs(graph.time - nsteps * dt) < 1e-15
    # checkpoint at step 10, restart, continue: bit-identical to the uninterrupted run
    import os
    import tempfile
    with tempfile.TemporaryDirectory() as tmp:
        part = DeviceRK4(og, dg.from_numpy(q0), dt).step(10)
        part.save(os.path.join(tmp, "ck.npz"))
        cont = DeviceRK4.restore(og, os.path.join(tmp, "ck.npz")).step(nsteps - 10)
        assert cont.nsteps == nsteps and np.array_equal(dg.to_numpy(cont.state), got_g)
        other = Op(make_dcoll(gpu, dim, order, n + 1, "periodic"), **kw)
        with pytest.raises(Exception):
            DeviceRK4.restore(other, os.path.join(tmp, "ck.npz"))
    assert np.array_equal(got_g, got_e)
    assert rel_err(got_g, ref) <= TOL_RK, rel_err(got_g, ref)
    assert gpu.launch_count > launches0


def test_graph_compiled_function_semantics(gpu):
    """actx.compile(f, graph=True): scalars stay arguments (a new value is a new graph, never a stale
    constant), shapes key the cache, results of consecutive calls do not alias, and an out-of-range
    gather inside a replayed graph is reported at the next check."""
    from paper_2512_17101_b200 import errors

    def f(x, a, idx):
        y = gpu.np.sqrt(x * x + a)
        return {"y": y, "picked": y[idx] * 2.0}

    cf = gpu.compile(f, graph=True)
    rng = np.random.default_rng(0)
    idx_h = np.array([3, 0, 7, 7, 2], dtype=np.int64)
    idx = gpu.from_numpy(idx_h)
    outs = []
    for call, a in enumerate([1.5, 1.5, 1.5, 2.5, 2.5, 2.5]):
        xh = rng.standard_normal(11)
        out = cf(gpu.from_numpy(xh), a, idx)
        ref = np.sqrt(xh * xh + a)
        assert np.array_equal(gpu.to_numpy(out["y"]), ref), (call, a)
        assert np.array_equal(gpu.to_numpy(out["picked"]), ref[idx_h] * 2.0)
        outs.append((out["y"], ref))
    for y, ref in outs:                                   # earlier results were not overwritten by later replays
        assert np.array_equal(gpu.to_numpy(y), ref)
    assert cf.replays == 4 and len(cf._graphs) == 2       # per scalar value: eager, capture + replay, replay
    bad = gpu.from_numpy(np.array([3, 0, 11, 7, 2], dtype=np.int64))
    out = cf(gpu.from_numpy(rng.standard_normal(11)), 1.5, bad)       # same signature: replayed, no host check ...
    with pytest.raises(errors.OutOfBoundsIndex):          # ... the device-side flag is raised at the next synchronisation
        gpu.to_numpy(out["picked"])
    ok = cf(gpu.from_numpy(np.ones(11)), 1.5, idx)        # the flag is cleared once reported
    assert np.array_equal(gpu.to_numpy(ok["y"]), np.sqrt(np.ones(11) + 1.5))


def test_edited_outlined_body_is_not_dispatched_by_name(gpu):
    """A function NAMED like a fused kernel but with a different body (here: another wave-speed estimate in
    the helpers of dg_euler_rhs) must not silently run the built-in physics: the context executes the body
    op by op on the device, and the result matches the oracle running the same edited body."""
    from paper_2512_17101_b200 import operators
    cpu = NumpyArrayContext()
    saved = operators._wavespeed
    try:
        def _wavespeed(actx, gamma, q, vel, p, dim):               # edited helper: a cruder bound
            return actx.np.sqrt(gamma * p / q[0]) * 2.0
        _wavespeed.__module__ = operators.__name__
        operators._wavespeed = _wavespeed
        dc, dg = make_dcoll(cpu, 3, 2, 3, "mixed"), make_dcoll(gpu, 3, 2, 3, "mixed")
        q0 = random_state(3, dc.nelements, dc.Np, seed=4)
        n_fused0 = gpu.launch_count
        with pytest.warns(RuntimeWarning, match="does not match the body"):
            og = EulerOperator(dg, farfield=FARFIELD[3])
        assert not getattr(og._f, "fused", False)
        ref = dc.to_numpy(EulerOperator(dc, farfield=FARFIELD[3]).rhs(dc.from_numpy(q0)))
        got = dg.to_numpy(og.rhs(dg.from_numpy(q0)))
        assert rel_err(got, ref) <= TOL_RHS
        assert gpu.launch_count - n_fused0 > 10                    # op by op, not one fused kernel
    finally:
        operators._wavespeed = saved
    # the unedited program dispatches to the fused kernel again and differs from the edited physics
    og2 = EulerOperator(dg, farfield=FARFIELD[3])
    assert getattr(og2._f, "fused", False)
    got2 = dg.to_numpy(og2.rhs(dg.from_numpy(q0)))
    assert rel_err(got2, ref) > 1e-6


def test_integration_stub_executes(gpu):
    """the reference-side ctypes binding (integration/laze_backend_b200.py) runs the
    CallSteps of dg_ns_flux / dg_ns_div on NumPy arrays exactly as the reference's interpreter would bind
    them, and reproduces the oracle."""
    import importlib.util
    import os
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "integration", "laze_backend_b200.py")
    spec = importlib.util.spec_from_file_location("laze_backend_b200", path)
    stub = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(stub)
    cpu = NumpyArrayContext()
    d = make_dcoll(cpu, 3, 3, 3, "mixed")
    op = NavierStokesOperator(d, farfield=FARFIELD[3], mu=2e-2)
    q0 = random_state(3, d.nelements, d.Np, seed=6)
    q = d.from_numpy(q0)
    T_ref = np.asarray(cpu.to_numpy(op.flux(q)))
    rhs_ref = d.to_numpy(op.rhs(q))
    host = lambda a: np.asarray(cpu.to_numpy(a))
    fargs = [q0] + [host(a) for a in op._flux_args()]
    T = stub.run_call_step_b200("dg_ns_flux", {f"_p{k}": a for k, a in enumerate(fargs)})["out"]
    assert rel_err(T, T_ref) <= TOL_RHS
    dargs = [q0, T] + [host(a) for a in op._div_args()]
    # the handle is keyed on the face-map arrays: hand the stub the same ndarrays for both calls
    dargs[9], dargs[10] = fargs[7], fargs[8]
    out = stub.run_call_step_b200("dg_ns_div", {f"_p{k}": a for k, a in enumerate(dargs)})["out"]
    assert rel_err(out, rhs_ref) <= TOL_RHS
    stub.close()
