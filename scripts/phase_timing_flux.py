"""Per-phase cycles of warp 0 of every CTA in k_nsflux3 / k_nsdiv3 (library built with -DDGB_PHASE_TIMING).
    python scripts/ab_variants.py --build timing   # builds libdgb200_timing.so
    DGB_LIB=.../libdgb200_timing.so python scripts/phase_timing_flux.py [n]
"""
import ctypes as C, sys
sys.path.insert(0, ".")
import numpy as np
from paper_2512_17101_b200 import B200ArrayContext, NavierStokesOperator
from paper_2512_17101_b200.fused import get_disc
from tests.common import make_dcoll, random_state
n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
actx = B200ArrayContext()
d = make_dcoll(actx, 3, 3, n, "periodic")
op = NavierStokesOperator(d, mu=1e-3)
q = d.from_numpy(random_state(3, d.nelements, d.Np))
for _ in range(3): op.rhs(q)
actx.synchronize()
disc = get_disc(actx, 3, q.data, 0, d.Sw, d.drdx, d.lift, d.normals, d.fscale, d.vmap_m, d.vmap_p, d.bc_kind)
out = (C.c_longlong * 8)()
def read():
    actx.synchronize(); actx.lib.dgb_debug_phase_cycles(disc.handle, out); return np.array(list(out), dtype=float)
read()
reps = 5
for _ in range(reps): T = op.flux(q)
v = read()
names = ["ticket + stage next + wait rows", "face averages (gathers)", "DMMA + combination", "pointwise flux + store"]
print("k_nsflux3, warp 0 of each CTA, share of its time per phase:")
for k in range(4): print(f"  {names[k]:34s} {100 * v[k] / v[:4].sum():5.1f} %   {v[k] / reps / 148 / 1.965e3:9.1f} us per CTA-warp and launch")
for _ in range(reps): op._div(q.data, T, *op._div_args())
v = read()
names = ["wait for q/lam/conn of this block", "face phase (gathers)", "wait T rows", "DMMA", "stage rows + store",
         "ticket + stage q/lam/conn of next block"]
print("k_nsdiv3:")
for k in (5, 0, 1, 2, 3, 4): print(f"  {names[k]:40s} {100 * v[k] / v[:6].sum():5.1f} %   {v[k] / reps / 148 / 1.965e3:9.1f} us per CTA-warp and launch")
