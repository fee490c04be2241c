"""Two ranks on one GPU with the peer-memory halo transport; each rank logs to gpurun_out/peer_<rank>.log."""
import os, sys, socket, traceback
sys.path.insert(0, ".")
import torch.multiprocessing as mp

def worker(rank, port):
    sys.stderr = sys.stdout = open(f"gpurun_out/peer_{rank}.log", "w", buffering=1)
    try:
        import numpy as np
        import torch.distributed as dist
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=2)
        from paper_2512_17101_b200 import B200ArrayContext, DGDiscretization, EulerOperator, NavierStokesOperator, box_mesh
        from paper_2512_17101_b200.dg.partition import interior_first, partition_elements, rank_mesh
        from paper_2512_17101_b200.halo import HaloExchange, TorchCommunicator
        from tests.common import random_state
        actx = B200ArrayContext()
        base = box_mesh((3,) * 3, (-1,) * 3, (1,) * 3, periodic=(True,) * 3)
        part = partition_elements(base, 2)
        local, plan = interior_first(*rank_mesh(base, part, rank))
        q0 = random_state(3, base.nelements, 10, seed=9)[:, plan.global_ids, :]
        d = DGDiscretization(actx, local, 2, ghost_elements=plan.nghost)
        halo = HaloExchange(actx, plan, TorchCommunicator(), d.Np, transport="peer")
        print("setup done", flush=True)
        e = d.to_numpy(halo.euler_rhs(EulerOperator(d), d.from_numpy(q0)))
        print("euler done", float(np.abs(e).max()), flush=True)
        v = d.to_numpy(halo.ns_rhs(NavierStokesOperator(d, mu=2e-2), d.from_numpy(q0)))
        print("ns done", float(np.abs(v).max()), flush=True)
        dist.destroy_process_group()
    except Exception:
        traceback.print_exc()

if __name__ == "__main__":
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    ps = [ctx.Process(target=worker, args=(r, port)) for r in range(2)]
    for p in ps: p.start()
    for p in ps: p.join(timeout=90)
    for p in ps:
        if p.is_alive():
            print("rank still alive after 90 s: killing"); p.kill(); p.join(10)
