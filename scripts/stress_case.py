"""Stress helper: repeat small parity cases many times and report any mismatch (flakiness hunt)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle.laze_port import NumpyArrayContext, rel_err
from paper_2512_17101_b200 import B200ArrayContext, EulerOperator, NavierStokesOperator
from tests.common import FARFIELD, make_dcoll, random_state, smooth_state

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
cases = [(2, 2, 5, "periodic"), (2, 3, 4, "mixed"), (3, 3, 3, "periodic"), (3, 2, 3, "mixed"), (2, 1, 3, "farfield")]
gpu, cpu = B200ArrayContext(), NumpyArrayContext()
nbad = 0
for it in range(reps):
    for dim, order, n, bc in cases:
        dc, dg = make_dcoll(cpu, dim, order, n, bc), make_dcoll(gpu, dim, order, n, bc)
        q0 = random_state(dim, dc.nelements, dc.Np, seed=it)
        for Op, kw in [(EulerOperator, {}), (NavierStokesOperator, {"mu": 2e-2})]:
            oc, og = Op(dc, farfield=FARFIELD[dim], **kw), Op(dg, farfield=FARFIELD[dim], **kw)
            ref = dc.to_numpy(oc.rhs(dc.from_numpy(q0)))
            got = dg.to_numpy(og.rhs(dg.from_numpy(q0)))
            e = rel_err(got, ref)
            if not e < 1e-12:
                nbad += 1
                err = np.abs(got - ref)
                bad = np.argwhere(err > 1e-10 * max(1, np.abs(ref).max()))
                print("MISMATCH", it, (dim, order, n, bc), Op.__name__, e, "elems", sorted(set(bad[:, 1].tolist()))[:12],
                      "fields", sorted(set(bad[:, 0].tolist())), "nodes", sorted(set(bad[:, 2].tolist())), flush=True)
print("done reps", reps, "mismatches", nbad)
