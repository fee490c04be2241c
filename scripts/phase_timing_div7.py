"""Per-phase cycles of consumer warp 0 and producer warp 4 of every CTA in k_nsdiv7 (library built with
-DDGB_PHASE_TIMING -DDGB_DIV_KERNEL_DEFAULT=7):  DGB_LIB=.../libdgb200_timing7.so python scripts/phase_timing_div7.py [n]"""
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
T = op.flux(q)
read()
reps = 5
for _ in range(reps): op._div(q.data, T, *op._div_args())
v = read()
names = ["consumer: wait for a full stage", "consumer: contraction + result store", "producer: stage T rows, ticket, wait small inputs",
         "producer: face phase (gathers)", "producer: stage next small inputs, wait T rows, hand over",
         "producer: wait for the consumer", "producer: 1/J + epilogue store"]
print("k_nsdiv7, consumer warp 0 / producer warp 4 of each CTA:")
for k in range(7):
    tot = v[:2].sum() if k < 2 else v[2:7].sum()
    print(f"  {names[k]:60s} {100 * v[k] / tot:5.1f} %   {v[k] / reps / 148 / 1.965e3:9.1f} us per warp and launch")
