"""Per-field error of the fused multi-species right-hand side against the oracle and against the op-by-op device path."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle.laze_port import NumpyArrayContext
from paper_2512_17101_b200 import B200ArrayContext, Mixture, MultispeciesOperator
from tests.common import make_dcoll
from tests.test_multispecies import ms_state
gpu, cpu = B200ArrayContext(), NumpyArrayContext()
for order, n, bc in [(3, 6, "periodic"), (3, 10, "periodic"), (3, 12, "farfield"), (2, 10, "periodic")]:
    dc, dg = make_dcoll(cpu, 3, order, n, bc), make_dcoll(gpu, 3, order, n, bc)
    oc, og = MultispeciesOperator(dc, Mixture()), MultispeciesOperator(dg, Mixture())
    gen = MultispeciesOperator(dg, Mixture(), fused=False, graph=False)
    q0 = ms_state(oc, dc.nodes())
    ref = dc.to_numpy(oc.rhs(dc.from_numpy(q0)))
    got = dg.to_numpy(og.rhs(dg.from_numpy(q0)))
    got2 = dg.to_numpy(gen.rhs(dg.from_numpy(q0)))
    Tref = np.asarray(oc.flux(dc.from_numpy(q0).data, None)) if False else None
    e1 = np.abs(got - ref).max(axis=(1, 2)); e2 = np.abs(got2 - ref).max(axis=(1, 2))
    print(f"p{order} n={n} {bc}: max|ref| {np.abs(ref).max():.3f}")
    print("   fused   - oracle per field:", " ".join(f"{v:.1e}" for v in e1))
    print("   generic - oracle per field:", " ".join(f"{v:.1e}" for v in e2))
