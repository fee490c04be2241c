"""Per-phase wall-clock split of the fused kernels (needs libdgb200_timing.so; DGB_LIB selects it)."""
import sys, os, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2512_17101_b200 import B200ArrayContext, DGDiscretization, NavierStokesOperator, box_mesh
from paper_2512_17101_b200.fused import get_disc
n = int(sys.argv[1]) if len(sys.argv) > 1 else 48
actx = B200ArrayContext()
mesh = box_mesh((n,) * 3, (-1.,) * 3, (1.,) * 3, periodic=(True,) * 3)
d = DGDiscretization(actx, mesh, 3)
op = NavierStokesOperator(d, mu=1e-3)
rng = np.random.default_rng(0)
q0 = np.empty((5, d.nelements, 20)); q0[0] = rng.uniform(.9, 1.1, q0[0].shape); q0[2:] = rng.uniform(-.1, .1, q0[2:].shape); q0[1] = 2.5 + rng.uniform(0, .1, q0[0].shape)
q = d.from_numpy(q0)
for _ in range(3): op.rhs(q)
actx.synchronize()
disc = get_disc(actx, 3, q.data, 0, d.Sw, d.drdx, d.lift, d.normals, d.fscale, d.vmap_m, d.vmap_p, d.bc_kind)
out = (C.c_longlong * 8)()
actx.lib.dgb_debug_phase_cycles(disc.handle, out)
for _ in range(5): op.rhs(q)
actx.synchronize()
actx.lib.dgb_debug_phase_cycles(disc.handle, out)
v = np.array(list(out), dtype=float)
names = ["rhs:geo", "rhs:phase1", "rhs:phase2", "rhs:phase3", "grad:stage", "grad:qstar", "grad:mma+store", "-"]
tr, tg = v[:4].sum(), v[4:7].sum()
for k in range(7):
    print(f"{names[k]:16s} {v[k]:.3e} cycles  {100 * v[k] / (tr if k < 4 else tg):5.1f}%")
