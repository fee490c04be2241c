"""One RK4 step of DeviceRK4 (graph) on the 3D NS p3 operator at a given size: ms per step and per stage."""
import sys, time
sys.path.insert(0, ".")
from paper_2512_17101_b200 import B200ArrayContext, DeviceRK4, NavierStokesOperator
from tests.common import make_dcoll, smooth_state
n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
actx = B200ArrayContext()
d = make_dcoll(actx, 3, 3, n, "periodic")
op = NavierStokesOperator(d, mu=1e-2)
g = DeviceRK4(op, d.from_numpy(smooth_state(d.nodes())), 1e-5, use_graph=True)
for _ in range(3): g.step()
actx.synchronize()
t0 = time.perf_counter()
for _ in range(20): g.step()
actx.synchronize()
ms = (time.perf_counter() - t0) / 20 * 1e3
print(f"n={n} {d.nelements * d.Np / 1e6:.2f} MDOF: {ms:.3f} ms per RK4 step, {ms / 4:.3f} ms per stage", flush=True)
