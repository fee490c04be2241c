"""The N>1 path on CPU: world_size-2 `gloo` process groups run the partition-aware right-hand side
(halo pack -> batched isend/irecv -> ghost arrays) with the oracle context and must reproduce the
single-domain result."""
import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, mode, outq, device=False, transport="nccl"):
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2512_17101_b200 import DGDiscretization, EulerOperator, NavierStokesOperator, box_mesh
        from paper_2512_17101_b200.dg.partition import interior_first, partition_elements, rank_mesh, ring_slab
        from paper_2512_17101_b200.halo import HaloExchange, TorchCommunicator
        from tests.common import random_state
        if device:        # both ranks share cuda:0; gloo stages the payloads through the host
            from paper_2512_17101_b200 import B200ArrayContext
            actx = B200ArrayContext()
        else:
            from oracle.laze_port import NumpyArrayContext
            actx = NumpyArrayContext()
        comm = TorchCommunicator()
        base = box_mesh((3,) * 3, (-1,) * 3, (1,) * 3, periodic=(True,) * 3)
        if mode == "partition":
            part = partition_elements(base, world)
            local, plan = rank_mesh(base, part, rank)
            q0 = random_state(3, base.nelements, 10, seed=9)[:, plan.global_ids, :]
        else:
            local, plan = ring_slab(base, 3, rank, world, -1.0, 1.0)
            q0 = random_state(3, base.nelements, 10, seed=9 + rank)
        if device:
            local, plan2 = interior_first(local, plan)
            q0 = q0[:, plan2.local_perm, :]
            ids = plan2.global_ids if plan2.global_ids is not None else plan2.local_perm
            plan = plan2
        else:
            ids = plan.global_ids
        d = DGDiscretization(actx, local, 2, ghost_elements=plan.nghost)
        halo = HaloExchange(actx, plan, comm, d.Np, transport=transport)
        assert halo._can_overlap() == device
        e = d.to_numpy(halo.euler_rhs(EulerOperator(d), d.from_numpy(q0)))
        v = d.to_numpy(halo.ns_rhs(NavierStokesOperator(d, mu=2e-2), d.from_numpy(q0)))
        if device:      # the plain exchange-then-compute order gives the same bits, and so does a second evaluation
            v3 = d.to_numpy(halo.ns_rhs(NavierStokesOperator(d, mu=2e-2), d.from_numpy(q0)))
            assert np.array_equal(v, v3)
            halo.overlap = False
            v2 = d.to_numpy(halo.ns_rhs(NavierStokesOperator(d, mu=2e-2), d.from_numpy(q0)))
            assert np.array_equal(v, v2)
        halo.close()
        outq.put((rank, ids, e, v, halo.messages_per_exchange, halo.bytes_per_exchange))
    finally:
        dist.destroy_process_group()


def _run(mode, device=False, transport="nccl", world=2, target=None):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=target or _worker, args=(r, world, port, mode, q, device, transport)) for r in range(world)]
    for p in procs:
        p.start()
    try:
        res = sorted([q.get(timeout=240) for _ in procs], key=lambda t: t[0])
        for p in procs:
            p.join(timeout=60)
            assert p.exitcode == 0
    finally:
        for p in procs:          # never leave a worker (and its kernels) behind
            if p.is_alive():
                p.kill()
                p.join(timeout=10)
    return res


@pytest.mark.timeout(600)
@pytest.mark.parametrize("world", [2, 4, 8])
def test_partition_matches_single_domain(world):
    """Recursive-coordinate-bisection partitions over 2, 4 and 8 gloo ranks == the single-domain oracle."""
    sys.path.insert(0, ROOT)
    from oracle.laze_port import NumpyArrayContext, rel_err
    from paper_2512_17101_b200 import DGDiscretization, EulerOperator, NavierStokesOperator, box_mesh
    from tests.common import random_state
    res = _run("partition", world=world)
    actx = NumpyArrayContext()
    mesh = box_mesh((3,) * 3, (-1,) * 3, (1,) * 3, periodic=(True,) * 3)
    d = DGDiscretization(actx, mesh, 2)
    q0 = random_state(3, mesh.nelements, 10, seed=9)
    ref_e = d.to_numpy(EulerOperator(d).rhs(d.from_numpy(q0)))
    ref_v = d.to_numpy(NavierStokesOperator(d, mu=2e-2).rhs(d.from_numpy(q0)))
    full_e, full_v = np.empty_like(ref_e), np.empty_like(ref_v)
    for rank, ids, e, v, nmsg, nbytes in res:
        full_e[:, ids, :], full_v[:, ids, :] = e, v
        assert 1 <= nmsg <= world - 1 and nbytes > 0
    assert rel_err(full_e, ref_e) <= 1e-13 and rel_err(full_v, ref_v) <= 1e-13


@pytest.mark.timeout(600)
@pytest.mark.parametrize("world", [2, 4, 8])
def test_ring_matches_long_box(world):
    """`world` periodic boxes wired as a ring (bench.py's weak-scaling layout) == one (3*world)x3x3 periodic box."""
    sys.path.insert(0, ROOT)
    from oracle.laze_port import NumpyArrayContext, rel_err
    from paper_2512_17101_b200 import DGDiscretization, NavierStokesOperator, box_mesh
    from tests.common import random_state
    res = _run("ring", world=world)
    actx = NumpyArrayContext()
    glob = box_mesh((3 * world, 3, 3), (-1, -1, -1), (2.0 * world - 1.0, 1, 1), periodic=(True,) * 3)
    base = box_mesh((3,) * 3, (-1,) * 3, (1,) * 3, periodic=(True,) * 3)
    d = DGDiscretization(actx, glob, 2)
    gkey = {tuple(np.round(c, 9)): e for e, c in enumerate(glob.vertices.mean(axis=1))}
    q0 = np.empty((5, glob.nelements, 10))
    idx = []
    for r in range(world):
        cent = base.vertices.mean(axis=1) + np.array([2.0 * r, 0, 0])
        idx.append(np.array([gkey[tuple(np.round(c, 9))] for c in cent]))
        q0[:, idx[r], :] = random_state(3, base.nelements, 10, seed=9 + r)
    ref = d.to_numpy(NavierStokesOperator(d, mu=2e-2).rhs(d.from_numpy(q0)))
    for rank, _, e, v, nmsg, nbytes in res:
        assert nmsg == 2
        assert rel_err(v, ref[:, idx[rank], :]) <= 1e-12


@pytest.mark.gpu
@pytest.mark.timeout(600)
def test_two_ranks_one_gpu_overlapped_exchange():
    """The device path of the N>1 run -- interior-first renumbering, element-range kernels, exchange on a
    communication stream overlapped with the interior range of each pass -- with two ranks sharing the
    one GPU of the test box (gloo stages the messages through the host; NCCL refuses two ranks per
    device).  Must reproduce the single-domain oracle and the non-overlapped order bit for bit."""
    sys.path.insert(0, ROOT)
    from oracle.laze_port import NumpyArrayContext, rel_err
    from paper_2512_17101_b200 import DGDiscretization, EulerOperator, NavierStokesOperator, box_mesh
    from tests.common import random_state
    actx = NumpyArrayContext()
    # partition of one periodic box
    res = _run("partition", device=True)
    mesh = box_mesh((3,) * 3, (-1,) * 3, (1,) * 3, periodic=(True,) * 3)
    d = DGDiscretization(actx, mesh, 2)
    q0 = random_state(3, mesh.nelements, 10, seed=9)
    ref_e = d.to_numpy(EulerOperator(d).rhs(d.from_numpy(q0)))
    ref_v = d.to_numpy(NavierStokesOperator(d, mu=2e-2).rhs(d.from_numpy(q0)))
    full_e, full_v = np.empty_like(ref_e), np.empty_like(ref_v)
    for rank, ids, e, v, nmsg, nbytes in res:
        full_e[:, ids, :], full_v[:, ids, :] = e, v
    assert rel_err(full_e, ref_e) <= 1e-12 and rel_err(full_v, ref_v) <= 1e-12
    # bench.py's ring of periodic boxes
    res = _run("ring", device=True)
    glob = box_mesh((6, 3, 3), (-1, -1, -1), (3, 1, 1), periodic=(True,) * 3)
    base = box_mesh((3,) * 3, (-1,) * 3, (1,) * 3, periodic=(True,) * 3)
    d = DGDiscretization(actx, glob, 2)
    gkey = {tuple(np.round(c, 9)): e for e, c in enumerate(glob.vertices.mean(axis=1))}
    q0 = np.empty((5, glob.nelements, 10))
    idx = []
    for r in range(2):
        cent = base.vertices.mean(axis=1) + np.array([2.0 * r, 0, 0])
        idx.append(np.array([gkey[tuple(np.round(c, 9))] for c in cent]))
        q0[:, idx[r], :] = random_state(3, base.nelements, 10, seed=9 + r)
    ref = d.to_numpy(NavierStokesOperator(d, mu=2e-2).rhs(d.from_numpy(q0)))
    for rank, perm, e, v, nmsg, nbytes in res:
        assert nmsg == 2
        assert rel_err(v, ref[:, idx[rank][perm], :]) <= 1e-12


@pytest.mark.gpu
@pytest.mark.timeout(600)
def test_two_ranks_one_gpu_peer_memory_transport():
    """transport="peer": the pack kernel of one rank stores the halo rows straight into the other rank's
    ghost array through CUDA-IPC mapped memory (the two processes share the one GPU of the test box; on
    a multi-GPU node the same mapping goes over NVLink), ordered by stream flags.  Same checks as above."""
    sys.path.insert(0, ROOT)
    from oracle.laze_port import NumpyArrayContext, rel_err
    from paper_2512_17101_b200 import DGDiscretization, EulerOperator, NavierStokesOperator, box_mesh
    from tests.common import random_state
    actx = NumpyArrayContext()
    res = _run("partition", device=True, transport="peer")
    mesh = box_mesh((3,) * 3, (-1,) * 3, (1,) * 3, periodic=(True,) * 3)
    d = DGDiscretization(actx, mesh, 2)
    q0 = random_state(3, mesh.nelements, 10, seed=9)
    ref_e = d.to_numpy(EulerOperator(d).rhs(d.from_numpy(q0)))
    ref_v = d.to_numpy(NavierStokesOperator(d, mu=2e-2).rhs(d.from_numpy(q0)))
    full_e, full_v = np.empty_like(ref_e), np.empty_like(ref_v)
    for rank, ids, e, v, nmsg, nbytes in res:
        full_e[:, ids, :], full_v[:, ids, :] = e, v
        assert nbytes > 0
    assert rel_err(full_e, ref_e) <= 1e-12 and rel_err(full_v, ref_v) <= 1e-12
    res = _run("ring", device=True, transport="peer")
    glob = box_mesh((6, 3, 3), (-1, -1, -1), (3, 1, 1), periodic=(True,) * 3)
    base = box_mesh((3,) * 3, (-1,) * 3, (1,) * 3, periodic=(True,) * 3)
    d = DGDiscretization(actx, glob, 2)
    gkey = {tuple(np.round(c, 9)): e for e, c in enumerate(glob.vertices.mean(axis=1))}
    q0 = np.empty((5, glob.nelements, 10))
    idx = []
    for r in range(2):
        cent = base.vertices.mean(axis=1) + np.array([2.0 * r, 0, 0])
        idx.append(np.array([gkey[tuple(np.round(c, 9))] for c in cent]))
        q0[:, idx[r], :] = random_state(3, base.nelements, 10, seed=9 + r)
    ref = d.to_numpy(NavierStokesOperator(d, mu=2e-2).rhs(d.from_numpy(q0)))
    for rank, perm, e, v, nmsg, nbytes in res:
        assert rel_err(v, ref[:, idx[rank][perm], :]) <= 1e-12


def _sendrecv_worker(rank, world, port, mode, outq, device=False, transport="nccl"):
    """actx.send / actx.receive of the reference surface (frontend.py:469-478) on the device context."""
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2512_17101_b200 import B200ArrayContext
        from paper_2512_17101_b200.halo import TorchCommunicator
        actx = B200ArrayContext(comm=TorchCommunicator())
        peer = 1 - rank
        x = actx.from_numpy(np.arange(12, dtype=np.float64).reshape(3, 4) + 100 * rank)
        k = actx.from_numpy(np.array([7, -3, 5], dtype=np.int64) * (rank + 1))
        # both ranks receive first and send afterwards: nothing is posted until a received array is used
        got_x = actx.receive(peer, 11, (3, 4))
        got_k = actx.receive(peer, 12, (3,), dtype=np.int64)
        y = actx.send(x * 2.0, peer, 11, stapled_to=x)
        actx.send(k, peer, 12, stapled_to=y)
        total = got_x + y                                   # first use: the batch goes out
        outq.put((rank, actx.to_numpy(total), actx.to_numpy(got_k), got_k.dtype == np.int64))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.timeout(300)
def test_context_send_receive_two_ranks():
    res = _run("sendrecv", device=True, target=_sendrecv_worker)
    for rank, total, got_k, is_i64 in res:
        peer = 1 - rank
        mine = np.arange(12, dtype=np.float64).reshape(3, 4) + 100 * rank
        theirs = np.arange(12, dtype=np.float64).reshape(3, 4) + 100 * peer
        assert np.array_equal(total, 2.0 * theirs + mine)
        assert is_i64 and np.array_equal(got_k, np.array([7, -3, 5]) * (peer + 1))


def _ms_worker(rank, world, port, mode, outq, device=False, transport="nccl"):
    """Multi-species operator through ``HaloExchange.ms_rhs`` (state halos, then flux-plane halos)."""
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2512_17101_b200 import DGDiscretization, Mixture, MultispeciesOperator, box_mesh
        from paper_2512_17101_b200.dg.partition import interior_first, partition_elements, rank_mesh
        from paper_2512_17101_b200.halo import HaloExchange, TorchCommunicator
        from oracle.laze_port import NumpyArrayContext
        from tests.test_multispecies import ms_state
        if device:
            from paper_2512_17101_b200 import B200ArrayContext
            actx = B200ArrayContext()
        else:
            actx = NumpyArrayContext()
        comm = TorchCommunicator()
        base = box_mesh((3,) * 3, (-1,) * 3, (1,) * 3, periodic=(True,) * 3)
        cpu = NumpyArrayContext()
        dref = DGDiscretization(cpu, base, 2)
        q0 = ms_state(MultispeciesOperator(dref, Mixture()), dref.nodes())
        local, plan = rank_mesh(base, partition_elements(base, world), rank)
        q0 = q0[:, plan.global_ids, :]
        if device:
            local, plan = interior_first(local, plan)
            q0 = q0[:, plan.local_perm, :]
        d = DGDiscretization(actx, local, 2, ghost_elements=plan.nghost)
        op = MultispeciesOperator(d, Mixture())
        halo = HaloExchange(actx, plan, comm, d.Np, transport=transport)
        v = d.to_numpy(halo.ms_rhs(op, d.from_numpy(q0)))
        if device:      # overlapped == exchange-then-compute, bit for bit; a second evaluation reuses the channels
            assert halo._can_overlap() and op._flux.fused and op._div.fused
            assert np.array_equal(v, d.to_numpy(halo.ms_rhs(op, d.from_numpy(q0))))
            halo.overlap = False
            assert np.array_equal(v, d.to_numpy(halo.ms_rhs(op, d.from_numpy(q0))))
        halo.close()
        outq.put((rank, plan.global_ids, v))
    finally:
        dist.destroy_process_group()


def _check_ms(res):
    from oracle.laze_port import NumpyArrayContext, rel_err
    from paper_2512_17101_b200 import DGDiscretization, Mixture, MultispeciesOperator, box_mesh
    from tests.test_multispecies import ms_state
    actx = NumpyArrayContext()
    mesh = box_mesh((3,) * 3, (-1,) * 3, (1,) * 3, periodic=(True,) * 3)
    d = DGDiscretization(actx, mesh, 2)
    op = MultispeciesOperator(d, Mixture())
    q0 = ms_state(op, d.nodes())
    ref = d.to_numpy(op.rhs(d.from_numpy(q0)))
    full = np.empty_like(ref)
    for rank, ids, v in res:
        full[:, ids, :] = v
    return rel_err(full, ref)


@pytest.mark.timeout(600)
@pytest.mark.parametrize("world", [2, 4])
def test_multispecies_partition_matches_single_domain(world):
    """BASELINE configs[4] is a multi-GPU config: the multi-species operator over 2 and 4 gloo ranks == single domain."""
    sys.path.insert(0, ROOT)
    assert _check_ms(_run("partition", world=world, target=_ms_worker)) <= 1e-13


@pytest.mark.gpu
@pytest.mark.timeout(600)
@pytest.mark.parametrize("transport", ["nccl", "peer"])
def test_two_ranks_one_gpu_multispecies(transport):
    """Fused multi-species kernels on element sub-ranges, both exchanges overlapped with the interior range of their
    pass, two ranks sharing the one GPU (gloo staging / CUDA-IPC peer stores)."""
    sys.path.insert(0, ROOT)
    assert _check_ms(_run("partition", device=True, transport=transport, target=_ms_worker)) <= 1e-12


def _rk_worker(rank, world, port, mode, outq, device=False, transport="nccl"):
    """A few RK4 steps on a partitioned mesh with the stage update fused into pass 2 (``HaloExchange.ns_rhs_rk``)."""
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2512_17101_b200 import DGDiscretization, NavierStokesOperator, box_mesh, rk4_step, rk4_step_fused
        from paper_2512_17101_b200.dg.partition import interior_first, partition_elements, rank_mesh
        from paper_2512_17101_b200.halo import HaloExchange, PartitionedOperator, TorchCommunicator
        from oracle.laze_port import NumpyArrayContext
        from tests.common import smooth_state
        if device:
            from paper_2512_17101_b200 import B200ArrayContext
            actx = B200ArrayContext()
        else:
            actx = NumpyArrayContext()
        comm = TorchCommunicator()
        base = box_mesh((3,) * 3, (-1,) * 3, (1,) * 3, periodic=(True,) * 3)
        dref = DGDiscretization(NumpyArrayContext(), base, 2)
        q0 = smooth_state(dref.nodes())
        local, plan = rank_mesh(base, partition_elements(base, world), rank)
        q0 = q0[:, plan.global_ids, :]
        if device:
            local, plan = interior_first(local, plan)
            q0 = q0[:, plan.local_perm, :]
        d = DGDiscretization(actx, local, 2, ghost_elements=plan.nghost)
        halo = HaloExchange(actx, plan, comm, d.Np, transport=transport)
        pop = PartitionedOperator(halo, NavierStokesOperator(d, mu=2e-2))
        qf, qu, t, dt = d.from_numpy(q0), d.from_numpy(q0), 0.0, 2e-3
        for _ in range(4):
            qf = rk4_step_fused(pop, qf, t, dt)
            qu = rk4_step(pop.rhs, qu, t, dt)
            t += dt
        halo.close()
        outq.put((rank, plan.global_ids, d.to_numpy(qf), d.to_numpy(qu)))
    finally:
        dist.destroy_process_group()


def _check_rk(res):
    from oracle.laze_port import NumpyArrayContext, rel_err
    from paper_2512_17101_b200 import DGDiscretization, NavierStokesOperator, box_mesh, rk4_step
    from tests.common import smooth_state
    actx = NumpyArrayContext()
    mesh = box_mesh((3,) * 3, (-1,) * 3, (1,) * 3, periodic=(True,) * 3)
    d = DGDiscretization(actx, mesh, 2)
    op = NavierStokesOperator(d, mu=2e-2)
    q, t, dt = d.from_numpy(smooth_state(d.nodes())), 0.0, 2e-3
    for _ in range(4):
        q = rk4_step(op.rhs, q, t, dt)
        t += dt
    ref = d.to_numpy(q)
    fused_, plain = np.empty_like(ref), np.empty_like(ref)
    for rank, ids, qf, qu in res:
        fused_[:, ids, :], plain[:, ids, :] = qf, qu
    return rel_err(fused_, ref), rel_err(plain, ref)


@pytest.mark.timeout(600)
def test_partitioned_fused_rk_matches_single_domain():
    """rk4_step_fused over a PartitionedOperator (2 gloo ranks, oracle context) == single-domain rk4_step."""
    sys.path.insert(0, ROOT)
    ef, eu = _check_rk(_run("partition", world=2, target=_rk_worker))
    assert ef <= 1e-13 and eu <= 1e-13


@pytest.mark.gpu
@pytest.mark.timeout(600)
@pytest.mark.parametrize("transport", ["nccl", "peer"])
def test_two_ranks_one_gpu_fused_rk(transport):
    """The same on the device: dgb_ns_div_rk_range on the interior and boundary ranges, both exchanges overlapped."""
    sys.path.insert(0, ROOT)
    ef, eu = _check_rk(_run("partition", device=True, transport=transport, target=_rk_worker))
    assert ef <= 1e-12 and eu <= 1e-12
