"""Throughput of the (unfused) multispecies RHS on B200 through the generic device ops, next to the fused NS RHS."""
import sys, time
sys.path.insert(0, ".")
from paper_2512_17101_b200 import B200ArrayContext, Mixture, MultispeciesOperator, NavierStokesOperator
from tests.common import make_dcoll, smooth_state
from tests.test_multispecies import ms_state
actx = B200ArrayContext()
print("| n | node-DOFs | fields | multispecies RHS ms, op by op | ms, one CUDA graph | MDOF/s (graph) | fused NS RHS ms |\n|---|---|---|---|---|---|---|")
for n in (8, 16, 24):
    d = make_dcoll(actx, 3, 3, n, "periodic")
    op = MultispeciesOperator(d, Mixture(), graph=True)
    op_eager = MultispeciesOperator(d, Mixture(), graph=False)
    q = d.from_numpy(ms_state(op, d.nodes()))
    ns_op = NavierStokesOperator(d, mu=1e-2)
    q5 = d.from_numpy(smooth_state(d.nodes()))
    def timed(fn, reps=5):
        fn(); fn(); fn(); actx.synchronize()          # eager call, capture call, first replay
        l0 = actx.launch_count; t0 = time.perf_counter()
        for _ in range(reps): fn()
        actx.synchronize()
        return (time.perf_counter() - t0) / reps * 1e3, (actx.launch_count - l0) // reps
    te, le = timed(lambda: op_eager.rhs(q))
    tm, lm = timed(lambda: op.rhs(q))
    tn, _ = timed(lambda: ns_op.rhs(q5))
    N = d.nelements * d.Np
    print(f"| {n} | {N} | {op.ncomp} | {te:.2f} ({le} launches) | {tm:.2f} | {N / tm / 1e3:.1f} | {tn:.3f} |", flush=True)
