"""Size-independent properties of the 3D NS p3 right-hand side at a size beyond the headline config
(default n=128: 12.58 M elements, 251.7 M DOFs, ~65 GB of arrays): free stream, conservation, reproducibility,
TMA-staged pass 2 == cp.async pass 2.  python scripts/large_case.py [n]"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_17101_b200 import B200ArrayContext, NavierStokesOperator  # noqa: E402
from tests.common import make_dcoll, smooth_state  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
gpu = B200ArrayContext()
t0 = time.time()
d = make_dcoll(gpu, 3, 3, n, "periodic")
E, Np = d.nelements, d.Np
print(f"n={n}: {E} elements, {E * Np} DOFs, mesh + discretisation {time.time() - t0:.1f} s", flush=True)
op = NavierStokesOperator(d, mu=1e-3)
qf = np.array([1.2, 2.9, 0.3, -0.2, 0.1])
qc = d.from_numpy(np.broadcast_to(qf[:, None, None], (5, E, Np)))
fs = d.norm_inf(op.rhs(qc))
print("free stream |rhs|_inf", fs, flush=True)
del qc
q = d.from_numpy(smooth_state(d.nodes()))
os.environ["DGB_DIV_KERNEL"] = "8"
r = op.rhs(q)
gpu.synchronize()
t1 = time.time()
for _ in range(5):
    r = op.rhs(q)
gpu.synchronize()
ms = (time.time() - t1) / 5 * 1e3
print(f"rhs {ms:.2f} ms = {E * Np / ms / 1e6:.2f} GDOF/s", flush=True)
rh = d.to_numpy(r)
w = np.einsum("i,ij->j", np.ones(Np), d.element.mass)
total = np.einsum("cej,j,e->c", rh, w, d.geo.jac)
scale = np.einsum("cej,j,e->c", np.abs(rh), w, d.geo.jac)
print("conservation |sum| / sum|.|", np.abs(total) / np.maximum(scale, 1.0), flush=True)
same = np.array_equal(d.to_numpy(op.rhs(q)), rh)
os.environ["DGB_DIV_KERNEL"] = "3"
same3 = np.array_equal(d.to_numpy(op.rhs(q)), rh)
print("reproducible", same, " k_nsdiv8 == k_nsdiv3", same3, " finite", bool(np.all(np.isfinite(rh))))
ok = fs < 5e-11 and same and same3 and np.all(np.abs(total) <= 1e-12 * np.maximum(scale, 1.0))
print("OK" if ok else "FAIL")
sys.exit(0 if ok else 1)
