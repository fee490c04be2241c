"""Steps per second of one RK4 step of the 3D NS p3 operator on small meshes: array-context RK4
(rk4_step), stage-fused RK4 (rk4_step_fused), DeviceRK4 without and with the CUDA graph."""
import sys, time
sys.path.insert(0, ".")
import numpy as np
from paper_2512_17101_b200 import B200ArrayContext, DeviceRK4, NavierStokesOperator, rk4_step, rk4_step_fused
from tests.common import make_dcoll, smooth_state
actx = B200ArrayContext()
print("| n | DOFs | rk4_step ms | rk4_step_fused ms | DeviceRK4 eager ms | DeviceRK4 graph ms |\n|---|---|---|---|---|---|")
for n in (4, 8, 16, 32, 64):
    d = make_dcoll(actx, 3, 3, n, "periodic")
    op = NavierStokesOperator(d, mu=1e-2)
    q0 = d.from_numpy(smooth_state(d.nodes()))
    dt, reps = 1e-4, 20
    def timed(fn):
        fn(); actx.synchronize()
        t0 = time.perf_counter()
        for _ in range(reps): fn()
        actx.synchronize()
        return (time.perf_counter() - t0) / reps * 1e3
    state = {"q": q0}
    def a(): state["q"] = rk4_step(op.rhs, state["q"], 0.0, dt)
    ta = timed(a)
    state["q"] = q0
    def b(): state["q"] = rk4_step_fused(op, state["q"], 0.0, dt)
    tb = timed(b)
    e = DeviceRK4(op, q0, dt, use_graph=False); te = timed(lambda: e.step())
    g = DeviceRK4(op, q0, dt, use_graph=True); tg = timed(lambda: g.step())
    print(f"| {n} | {d.nelements * d.Np} | {ta:.3f} | {tb:.3f} | {te:.3f} | {tg:.3f} |", flush=True)
