"""Debug helper: per-field / per-element parity errors of one (dim, order, n, bc) case."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle.laze_port import NumpyArrayContext, rel_err
from paper_2512_17101_b200 import B200ArrayContext, EulerOperator, NavierStokesOperator
from tests.common import FARFIELD, make_dcoll, random_state, smooth_state

dim, order, n, bc = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
gpu, cpu = B200ArrayContext(), NumpyArrayContext()
dc, dg = make_dcoll(cpu, dim, order, n, bc), make_dcoll(gpu, dim, order, n, bc)
for name, q0 in [("random", random_state(dim, dc.nelements, dc.Np, seed=1)), ("smooth", smooth_state(dc.nodes()))]:
    for Op, kw in [(EulerOperator, {}), (NavierStokesOperator, {"mu": 2e-2})]:
        oc, og = Op(dc, farfield=FARFIELD[dim], **kw), Op(dg, farfield=FARFIELD[dim], **kw)
        for rep in range(3):
            ref = dc.to_numpy(oc.rhs(dc.from_numpy(q0)))
            got = dg.to_numpy(og.rhs(dg.from_numpy(q0)))
            err = np.abs(got - ref)
            bad = np.argwhere(err > 1e-10 * max(1, np.abs(ref).max()))
            print(name, Op.__name__, rep, "rel", rel_err(got, ref), "nbad", len(bad),
                  "bad elems", sorted(set(bad[:, 1].tolist()))[:20], "bad fields", sorted(set(bad[:, 0].tolist())),
                  "bad nodes", sorted(set(bad[:, 2].tolist())))
        if Op is NavierStokesOperator:
            gref = dc.to_numpy(oc.grad(dc.from_numpy(q0))); ggot = dg.to_numpy(og.grad(dg.from_numpy(q0)))
            print("   grad rel", rel_err(ggot, gref))
