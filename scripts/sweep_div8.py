"""Randomised sweep: TMA-staged pass 2 (k_nsdiv8) against the cp.async pass 2 (k_nsdiv3), bitwise, over many
(dim, order, cells, boundary, state seed) combinations incl. ragged last blocks; and both against the oracle at 1e-12
for the small ones.  Run on the GPU box:  python scripts/sweep_div8.py [ncases]"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle.laze_port import NumpyArrayContext, rel_err  # noqa: E402
from paper_2512_17101_b200 import B200ArrayContext  # noqa: E402
from paper_2512_17101_b200.operators import NavierStokesOperator  # noqa: E402
from tests.common import FARFIELD, make_dcoll, random_state  # noqa: E402

ncases = int(sys.argv[1]) if len(sys.argv) > 1 else 40
rng = np.random.default_rng(20251217)
gpu, cpu = B200ArrayContext(), NumpyArrayContext()
bad = 0
for case in range(ncases):
    dim = int(rng.integers(2, 4))
    order = int(rng.integers(1, 5))
    n = int(rng.integers(3, 9 if dim == 3 else 14))
    bc = ["periodic", "mixed", "farfield"][int(rng.integers(0, 3))]
    seed = int(rng.integers(0, 1000))
    d = make_dcoll(gpu, dim, order, n, bc)
    op = NavierStokesOperator(d, farfield=FARFIELD[dim], mu=2e-2)
    q0 = random_state(dim, d.nelements, d.Np, seed=seed)
    q = d.from_numpy(q0)
    outs = {}
    for k in ("3", "8"):
        os.environ["DGB_DIV_KERNEL"] = k
        o1, o2 = op.rhs_rk(q, q, q, (1.0, 0.25, 0.5, -2.0))
        outs[k] = (d.to_numpy(op.rhs(q)), d.to_numpy(o1), d.to_numpy(o2))
    same = all(np.array_equal(a, b) for a, b in zip(outs["3"], outs["8"]))
    err = ""
    if d.nelements * d.Np <= 60000:
        dc = make_dcoll(cpu, dim, order, n, bc)
        ref = dc.to_numpy(NavierStokesOperator(dc, farfield=FARFIELD[dim], mu=2e-2).rhs(dc.from_numpy(q0)))
        e = rel_err(outs["8"][0], ref)
        err = f" oracle {e:.1e}"
        same = same and e <= 1e-12
    bad += not same
    print(f"{case:3d} dim {dim} p{order} n {n:2d} {bc:8s} E {d.nelements:6d}: {'OK' if same else 'FAIL'}{err}", flush=True)
print("failures:", bad)
sys.exit(1 if bad else 0)
