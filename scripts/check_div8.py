"""k_nsdiv8 (TMA-staged pass 2) against k_nsdiv3 on the same inputs: bitwise equality at several sizes,
then timings of both (CUDA events).  Run on the GPU box."""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2512_17101_b200 import B200ArrayContext  # noqa: E402
from paper_2512_17101_b200.operators import NavierStokesOperator  # noqa: E402
from tests.common import FARFIELD, make_dcoll, random_state  # noqa: E402

gpu = B200ArrayContext()
ok = True
cases = [(3, 3, 2, "mixed"), (3, 3, 5, "periodic"), (3, 3, 24, "mixed"), (3, 4, 8, "mixed"), (3, 2, 6, "periodic"),
         (3, 1, 6, "mixed"), (2, 3, 12, "mixed"), (2, 4, 9, "periodic"), (2, 1, 7, "farfield"), (2, 2, 8, "mixed")]
if "--quick" in sys.argv:
    cases = cases[:3]
for dim, order, n, bc in cases:
    d = make_dcoll(gpu, dim, order, n, bc)
    op = NavierStokesOperator(d, farfield=FARFIELD[dim], mu=2e-2)
    q = d.from_numpy(random_state(dim, d.nelements, d.Np, seed=3))
    outs = {}
    for k in ("3", "8"):
        os.environ["DGB_DIV_KERNEL"] = k
        outs[k] = d.to_numpy(op.rhs(q))
        o1, o2 = op.rhs_rk(q, q, q, (1.0, 0.25, 0.5, -2.0))
        outs[k + "rk"] = np.stack([d.to_numpy(o1), d.to_numpy(o2)])
    same = np.array_equal(outs["3"], outs["8"]) and np.array_equal(outs["3rk"], outs["8rk"])
    err = np.abs(outs["3"] - outs["8"]).max()
    print(f"dim {dim} p{order} n {n} {bc}: bitwise {'OK' if same else 'DIFF'}  max|d| {err:.3e}  finite {np.isfinite(outs['8']).all()}", flush=True)
    ok &= same
n = int(sys.argv[sys.argv.index("--n") + 1]) if "--n" in sys.argv else 64
d = make_dcoll(gpu, 3, 3, n, "periodic")
op = NavierStokesOperator(d, mu=1e-3)
q = d.from_numpy(random_state(3, d.nelements, d.Np, seed=1))
T = op.flux(q)
for k in ("3", "8", "3", "8"):
    os.environ["DGB_DIV_KERNEL"] = k
    for _ in range(3):
        r = op.rhs(q)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    t0 = time.time()
    ev[0].record()
    for _ in range(10):
        r = op.rhs(q)
    ev[1].record()
    torch.cuda.synchronize()
    print(f"DGB_DIV_KERNEL={k}: n={n} {d.nelements * d.Np / 1e6:.2f} MDOF  {ev[0].elapsed_time(ev[1]) / 10:.3f} ms per RHS (both passes)", flush=True)
sys.exit(0 if ok else 1)
