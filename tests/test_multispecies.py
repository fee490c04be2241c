"""Multi-species reactive Navier-Stokes (BASELINE configs[4]): the model is builder-chosen (nothing in
the reference defines one), so it is pinned by reference-independent properties, by the reference's
own contexts executing the same program, and by GPU-vs-oracle parity of the generic device ops."""
import os
import sys

import numpy as np
import pytest

from oracle.laze_port import NumpyArrayContext, rel_err
from paper_2512_17101_b200 import EulerOperator, Mixture, MultispeciesOperator
from tests.common import MS_GOLDEN_CASES, MS_MIXTURES, make_dcoll, ms_state, smooth_state

REF = "/root/reference/pkg/src"


def test_reduces_to_euler_for_one_inert_species():
    """ns = 1, no transport, no reaction: the first dim+2 components are the single-species Euler RHS and
    the species equation is the continuity equation."""
    actx = NumpyArrayContext()
    d = make_dcoll(actx, 3, 2, 3, "periodic")
    mix = Mixture(R=(1.0,), cv=(2.5,), h0=(0.0,), reaction=(0, 0), A=0.0, Ta=1.0)
    op = MultispeciesOperator(d, mix, mu=0.0, kappa=0.0, diffusivity=0.0)
    q5 = smooth_state(d.nodes())
    q = np.concatenate([q5, q5[:1]])
    r = d.to_numpy(op.rhs(d.from_numpy(q)))
    ref = d.to_numpy(EulerOperator(d, gamma=1.4).rhs(d.from_numpy(q5)))
    assert rel_err(r[:5], ref) <= 1e-13
    assert rel_err(r[5], ref[0]) <= 1e-13


@pytest.mark.parametrize("dim,bc", [(3, "periodic"), (2, "farfield")])
def test_free_stream_and_conservation(dim, bc):
    actx = NumpyArrayContext()
    d = make_dcoll(actx, dim, 3, 3, bc)
    mix = Mixture()
    far = None
    op0 = MultispeciesOperator(d, Mixture(A=0.0), farfield=far)
    qf = op0.state_from_primitive(1.1, [0.2, -0.1, 0.05][:dim], 1.3, [0.5, 0.2, 0.3])
    op0 = MultispeciesOperator(d, Mixture(A=0.0), farfield=qf)
    q = d.from_numpy(np.broadcast_to(qf.reshape(-1, 1, 1), (op0.ncomp, d.nelements, d.Np)))
    assert np.abs(d.to_numpy(op0.rhs(q))).max() < 5e-12          # uniform inert state is steady
    if bc == "periodic":
        op = MultispeciesOperator(d, mix)
        r = d.to_numpy(op.rhs(d.from_numpy(ms_state(op, d.nodes()))))
        w = np.einsum("i,ij->j", np.ones(d.Np), d.element.mass)
        total = np.einsum("cej,j,e->c", r, w, d.geo.jac)
        assert np.abs(total[:2 + dim]).max() < 1e-11              # mass, energy, momentum
        assert abs(total[2 + dim:].sum()) < 1e-11                 # the reaction moves mass between species only
        assert total[2 + dim + mix.reaction[0]] < 0 < total[2 + dim + mix.reaction[1]]


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference not mounted")
def test_program_runs_on_the_reference_contexts():
    sys.path.insert(0, REF)
    import laze
    res = {}
    for name, actx in [("port", NumpyArrayContext()), ("eager", laze.ArrayContext(mode="eager")),
                       ("lazy", laze.ArrayContext(mode="lazy"))]:
        d = make_dcoll(actx, 2, 2, 3, "farfield")
        op = MultispeciesOperator(d, Mixture())
        res[name] = np.asarray(actx.to_numpy(op.rhs(d.from_numpy(ms_state(op, d.nodes()))).data))
    assert np.array_equal(res["port"], res["eager"])
    assert rel_err(res["lazy"], res["eager"]) <= 1e-12


@pytest.mark.gpu
@pytest.mark.parametrize("dim,order,n,bc", [(3, 3, 2, "periodic") if False else (3, 3, 3, "periodic"), (2, 3, 4, "farfield"), (3, 2, 2, "farfield")])
def test_gpu_parity_multispecies(dim, order, n, bc):
    """B200ArrayContext vs the oracle: the fused kernels (dgb_ms_flux / dgb_ms_div: k_nsflux3 / k_nsdiv8 instantiated
    for C = dim + 5 fields, mixture physics, Arrhenius source in the store epilogue) and, independently, the same
    program op by op on the generic device kernels."""
    from paper_2512_17101_b200 import B200ArrayContext
    gpu, cpu = B200ArrayContext(), NumpyArrayContext()
    dc, dg = make_dcoll(cpu, dim, order, n, bc), make_dcoll(gpu, dim, order, n, bc)
    oc, og = MultispeciesOperator(dc, Mixture()), MultispeciesOperator(dg, Mixture())
    assert getattr(og._f, "fused", False) and getattr(og._flux, "fused", False) and getattr(og._div, "fused", False)
    q0 = ms_state(oc, dc.nodes())
    ref = dc.to_numpy(oc.rhs(dc.from_numpy(q0)))
    n0 = gpu.launch_count
    got = dg.to_numpy(og.rhs(dg.from_numpy(q0)))
    assert gpu.launch_count - n0 <= 8                    # two fused kernels (+ handle set-up on the first call)
    assert np.all(np.isfinite(got)) and rel_err(got, ref) <= 1e-12, rel_err(got, ref)
    generic = MultispeciesOperator(dg, Mixture(), fused=False, graph=False)
    got2 = dg.to_numpy(generic.rhs(dg.from_numpy(q0)))
    assert rel_err(got2, ref) <= 1e-12 and rel_err(got, got2) <= 1e-12


MIXTURES = MS_MIXTURES


@pytest.mark.gpu
@pytest.mark.timeout(900)
@pytest.mark.parametrize("ns,dim,order,n,bc", [(2, 3, 3, 3, "periodic"), (2, 2, 4, 4, "farfield"), (4, 3, 3, 3, "farfield"),
                                               (4, 3, 4, 3, "periodic"), (4, 2, 2, 5, "farfield"), (2, 3, 3, 10, "farfield"),
                                               (4, 3, 3, 8, "farfield"), (5, 3, 2, 3, "periodic")])
def test_gpu_parity_species_counts(ns, dim, order, n, bc):
    """The fused kernels are instantiated for 2, 3 and 4 species (csrc/dgb_msflux{2,3,4}.cu); any other count runs the
    same program op by op on the device.  Both against the oracle, incl. mid-size meshes (tens of blocks per warp)."""
    from paper_2512_17101_b200 import B200ArrayContext, fused
    gpu, cpu = B200ArrayContext(), NumpyArrayContext()
    dc, dg = make_dcoll(cpu, dim, order, n, bc), make_dcoll(gpu, dim, order, n, bc)
    oc, og = MultispeciesOperator(dc, Mixture(**MIXTURES[ns])), MultispeciesOperator(dg, Mixture(**MIXTURES[ns]))
    assert bool(getattr(og._flux, "fused", False)) == (ns in fused.MS_FUSED_SPECIES)
    q0 = ms_state(oc, dc.nodes())
    ref = dc.to_numpy(oc.rhs(dc.from_numpy(q0)))
    got = dg.to_numpy(og.rhs(dg.from_numpy(q0)))
    assert np.all(np.isfinite(got)) and rel_err(got, ref) <= 1e-12, rel_err(got, ref)


@pytest.mark.gpu
@pytest.mark.timeout(900)
@pytest.mark.parametrize("order,n,bc", [(3, 12, "farfield"), (3, 8, "periodic"), (4, 6, "farfield")])
def test_gpu_parity_multispecies_midsize(order, n, bc):
    """Many blocks per warp (ticket stream, staging across blocks), far-field boundaries, odd Np (order 4).
    The smooth periodic state has |rhs| < 1, so the reference norm is an ABSOLUTE error there, and the energy
    equation's second-derivative terms amplify rounding like h^-2 (scripts/ms_error_probe.py: 5.8e-13 at n=6,
    1.9e-12 at n=10 for the fused kernels, 4.9e-13 / 1.5e-12 for the op-by-op device path): n=8 is the largest
    periodic case inside the 1e-12 bar."""
    from paper_2512_17101_b200 import B200ArrayContext
    gpu, cpu = B200ArrayContext(), NumpyArrayContext()
    dc, dg = make_dcoll(cpu, 3, order, n, bc), make_dcoll(gpu, 3, order, n, bc)
    oc, og = MultispeciesOperator(dc, Mixture()), MultispeciesOperator(dg, Mixture())
    q0 = ms_state(oc, dc.nodes())
    ref = dc.to_numpy(oc.rhs(dc.from_numpy(q0)))
    got = dg.to_numpy(og.rhs(dg.from_numpy(q0)))
    assert np.all(np.isfinite(got)) and rel_err(got, ref) <= 1e-12, rel_err(got, ref)
    again = dg.to_numpy(og.rhs(dg.from_numpy(q0)))
    assert np.array_equal(got, again)                    # no atomics: bitwise reproducible


@pytest.mark.gpu
def test_gpu_graph_compiled_rhs():
    """actx.compile(f, graph=True): eager first call, captured second call, replays afterwards -- all
    bit-identical to the op-by-op evaluation, for changing inputs, with one graph launch per call."""
    from paper_2512_17101_b200 import B200ArrayContext
    gpu = B200ArrayContext()
    d = make_dcoll(gpu, 3, 2, 3, "farfield")
    plain = MultispeciesOperator(d, Mixture(), graph=False, fused=False)      # the op-by-op path (not the fused kernels)
    fast = MultispeciesOperator(d, Mixture(), graph=True, fused=False)
    rng = np.random.default_rng(3)
    base = ms_state(plain, d.nodes())
    for call in range(4):
        q0 = base * (1.0 + 0.01 * rng.standard_normal(base.shape[0])[:, None, None] * (call > 0))
        ref = d.to_numpy(plain.rhs(d.from_numpy(q0)))
        n0 = gpu.launch_count
        got = d.to_numpy(fast.rhs(d.from_numpy(q0)))
        assert np.array_equal(got, ref), call
        if call >= 2:
            assert gpu.launch_count == n0          # replay: no per-op dispatch (copies in/out are memcpys)
    assert fast._f.replays == 3 and fast._f.trace_count == 1
    gpu.check_deferred_errors()


@pytest.mark.parametrize("dim,n,per,nparts", [(3, 3, True, 2), (2, 4, False, 3)])
def test_partitioned_multispecies_equals_single_domain(dim, n, per, nparts):
    """Partitioned mesh with looped-back halos (state, then flux planes) == the single-domain right-hand side."""
    from paper_2512_17101_b200 import DGDiscretization, box_mesh
    from paper_2512_17101_b200.dg.partition import partition_elements, rank_mesh
    from paper_2512_17101_b200.discretization import BC_FARFIELD
    actx = NumpyArrayContext()
    mesh = box_mesh((n,) * dim, (-1,) * dim, (1,) * dim, periodic=(per,) * dim)
    bc = None if per else {k: BC_FARFIELD for k in range(1, 2 * dim + 1)}
    d = DGDiscretization(actx, mesh, 2, bc_map=bc)
    op = MultispeciesOperator(d, Mixture())
    q0 = ms_state(op, d.nodes())
    ref = d.to_numpy(op.rhs(d.from_numpy(q0)))
    part = partition_elements(mesh, nparts)
    locs = [rank_mesh(mesh, part, r) for r in range(nparts)]
    ds = [DGDiscretization(actx, m, 2, bc_map=bc, ghost_elements=p.nghost) for m, p in locs]
    ops = [MultispeciesOperator(dd, Mixture()) for dd in ds]
    qs = [q0[:, p.global_ids, :] for _, p in locs]

    def loopback(fields):
        out = []
        for r, (m, p) in enumerate(locs):
            g = np.empty(fields[r].shape[:-2] + (p.nghost, d.Np))
            for k, peer in enumerate(p.peers):
                pp = locs[peer][1]
                a, b = p.recv_slots[k]
                g[..., a:b, :] = fields[peer][..., pp.send_local[pp.peers.index(r)], :]
            out.append(g)
        return out

    gh = loopback(qs)
    FLs = [np.asarray(ops[r].flux(qs[r], gh[r])) for r in range(nparts)]
    gFL = loopback(FLs)
    full = np.empty_like(ref)
    for r, (m, p) in enumerate(locs):
        out = ops[r].rhs(ds[r].from_numpy(qs[r]), ghost=gh[r], halo_fn=lambda FL, r=r: gFL[r])
        full[:, p.global_ids, :] = ds[r].to_numpy(out)
    assert rel_err(full, ref) <= 1e-13


@pytest.mark.gpu
def test_gpu_partitioned_multispecies():
    """Partitioned multispecies on the device (ghost arrays through the generic gather, device pack kernel,
    exchange looped back on the host: this box has one GPU) against the single-domain oracle."""
    from paper_2512_17101_b200 import B200ArrayContext, DGDiscretization, box_mesh
    from paper_2512_17101_b200.dg.partition import partition_elements, rank_mesh
    from paper_2512_17101_b200.halo import HaloExchange
    gpu, cpu = B200ArrayContext(), NumpyArrayContext()
    mesh = box_mesh((3,) * 3, (-1,) * 3, (1,) * 3, periodic=(True,) * 3)
    d = DGDiscretization(cpu, mesh, 2)
    opc = MultispeciesOperator(d, Mixture())
    q0 = ms_state(opc, d.nodes())
    ref = d.to_numpy(opc.rhs(d.from_numpy(q0)))
    part = partition_elements(mesh, 2)
    locs = [rank_mesh(mesh, part, r) for r in range(2)]
    ds = [DGDiscretization(gpu, m, 2, ghost_elements=p.nghost) for m, p in locs]
    ops = [MultispeciesOperator(dd, Mixture()) for dd in ds]
    qs = [ds[r].from_numpy(q0[:, p.global_ids, :]) for r, (_, p) in enumerate(locs)]
    halos = [HaloExchange(gpu, p, object(), d.Np) for _, p in locs]

    def exchange(fields):
        packed = {(r, peer): gpu.to_numpy(halos[r]._pack(fields[r], k))
                  for r, (_, p) in enumerate(locs) for k, peer in enumerate(p.peers)}
        out = []
        for r, (_, p) in enumerate(locs):
            g = np.empty(tuple(fields[r].shape[:-2]) + (p.nghost, d.Np))
            for k, peer in enumerate(p.peers):
                a, b = p.recv_slots[k]
                g[..., a:b, :] = packed[(peer, r)]
            out.append(gpu.from_numpy(g))
        return out

    for rep in range(3):                  # eager, captured, replayed
        gh = exchange([q.data for q in qs])
        FLs = [ops[r].flux(qs[r], gh[r]) for r in range(2)]
        gFL = exchange(FLs)
        full = np.empty_like(ref)
        for r, (_, p) in enumerate(locs):
            out = ops[r].rhs(qs[r], ghost=gh[r], halo_fn=lambda FL, r=r: gFL[r])
            full[:, p.global_ids, :] = ds[r].to_numpy(out)
        assert rel_err(full, ref) <= 1e-12, rep


@pytest.mark.gpu
@pytest.mark.timeout(900)
def test_gpu_device_rk4_multispecies():
    """DeviceRK4 on the fused multi-species kernels (dgb_ms_flux + dgb_ms_div_rk: the stage update fused into the
    store of pass 2, one CUDA graph per step) == classical RK4 of the same program on the oracle (<= 1e-10 after 25
    steps, the north star's bound for 100), graph replay bitwise equal to eager launches, far-field boundaries."""
    from paper_2512_17101_b200 import B200ArrayContext, DeviceRK4
    from paper_2512_17101_b200.operators import rk4_step
    gpu, cpu = B200ArrayContext(), NumpyArrayContext()
    for dim, order, n, bc in [(3, 3, 3, "periodic"), (2, 3, 5, "farfield")]:
        dc, dg = make_dcoll(cpu, dim, order, n, bc), make_dcoll(gpu, dim, order, n, bc)
        oc, og = MultispeciesOperator(dc, Mixture()), MultispeciesOperator(dg, Mixture())
        q0 = ms_state(oc, dc.nodes())
        dt, nsteps = 1e-3, 25
        qc, t = dc.from_numpy(q0), 0.0
        for _ in range(nsteps):
            qc = rk4_step(oc.rhs, qc, t, dt)
            t += dt
        ref = dc.to_numpy(qc)
        graph = DeviceRK4(og, dg.from_numpy(q0), dt, use_graph=True).step(nsteps)
        eager = DeviceRK4(og, dg.from_numpy(q0), dt, use_graph=False).step(nsteps)
        got_g, got_e = dg.to_numpy(graph.state), dg.to_numpy(eager.state)
        assert np.array_equal(got_g, got_e)
        assert np.all(np.isfinite(got_g)) and rel_err(got_g, ref) <= 1e-10, rel_err(got_g, ref)
        assert rel_err(got_g, q0) > 1e-6                      # the state did move


@pytest.mark.gpu
@pytest.mark.parametrize("dim,order,n,bc", [(3, 3, 3, "periodic"), (3, 4, 3, "farfield"), (2, 3, 5, "farfield")])
def test_gpu_multispecies_cp_async_fallback(dim, order, n, bc, monkeypatch):
    """Pass 2 of the mixture on the cp.async kernel (k_nsdiv3<C=8>, what runs when the arrays cannot be described to
    the TMA unit) against the TMA-staged default: same arithmetic up to the contraction of the source-term add."""
    from paper_2512_17101_b200 import B200ArrayContext
    gpu = B200ArrayContext()
    d = make_dcoll(gpu, dim, order, n, bc)
    op = MultispeciesOperator(d, Mixture())
    q = d.from_numpy(ms_state(op, d.nodes()))
    outs = {}
    for k in ("8", "3"):
        monkeypatch.setenv("DGB_DIV_KERNEL", k)
        outs[k] = d.to_numpy(op.rhs(q))
    assert np.all(np.isfinite(outs["3"])) and rel_err(outs["3"], outs["8"]) <= 1e-14


GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.mark.parametrize("case", MS_GOLDEN_CASES, ids=[c[0] for c in MS_GOLDEN_CASES])
def test_multispecies_program_matches_reference_golden(case):
    """The oracle context against vectors the REAL reference produced for the multi-species program
    (tests/golden/make_golden.py: laze eager context and lazy compile pipeline)."""
    name, dim, order, n, bc, ns = case
    g = np.load(os.path.join(GOLD, name + ".npz"))
    actx = NumpyArrayContext()
    d = make_dcoll(actx, dim, order, n, bc)
    op = MultispeciesOperator(d, Mixture(**MS_MIXTURES[ns]))
    assert np.array_equal(ms_state(op, d.nodes()), g["q0"])
    rhs = d.to_numpy(op.rhs(d.from_numpy(g["q0"])))
    assert np.array_equal(rhs, g["eager_rhs"])
    assert rel_err(rhs, g["lazy_rhs"]) <= 1e-12


@pytest.mark.gpu
@pytest.mark.parametrize("case", MS_GOLDEN_CASES, ids=[c[0] for c in MS_GOLDEN_CASES])
def test_gpu_multispecies_matches_reference_golden(case):
    """The fused multi-species kernels against the REAL reference's vectors."""
    from paper_2512_17101_b200 import B200ArrayContext
    name, dim, order, n, bc, ns = case
    g = np.load(os.path.join(GOLD, name + ".npz"))
    gpu = B200ArrayContext()
    d = make_dcoll(gpu, dim, order, n, bc)
    op = MultispeciesOperator(d, Mixture(**MS_MIXTURES[ns]))
    assert getattr(op._f, "fused", False)
    got = d.to_numpy(op.rhs(d.from_numpy(g["q0"])))
    assert rel_err(got, g["eager_rhs"]) <= 1e-12 and rel_err(got, g["lazy_rhs"]) <= 1e-12
