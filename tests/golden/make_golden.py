"""Generate the golden vectors under tests/golden/ by running the DG operator program through the
REAL reference package (/root/reference/pkg/src/laze): its eager context, its lazy compile pipeline
(graph passes -> scalar IR -> loop passes -> NumPy interpreter) and its eager_eval oracle.

Run in the build container only (the reference does not travel to the GPU box):
    python tests/golden/make_golden.py [--ms-only]
Small cases only: the lazy interpreter runs at ~0.1 MDOF/s.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from paper_2512_17101_b200.operators import EulerOperator, NavierStokesOperator, rk4_step  # noqa: E402
from tests.common import FARFIELD, GOLDEN_CASES as CASES, make_dcoll, random_state, smooth_state  # noqa: E402


def run(actx, dim, order, n, bc, opname, kw, q0):
    d = make_dcoll(actx, dim, order, n, bc)
    op = (EulerOperator if opname == "euler" else NavierStokesOperator)(d, farfield=FARFIELD[dim], **kw)
    out = {"rhs": np.asarray(actx.to_numpy(op.rhs(d.from_numpy(q0)).data))}
    if opname == "ns":
        out["grad"] = np.asarray(actx.to_numpy(op.grad(d.from_numpy(q0)).data))
        out["rhs_grad_form"] = np.asarray(actx.to_numpy(op.rhs_grad_form(d.from_numpy(q0)).data))
        out["flux"] = np.asarray(actx.to_numpy(op.flux(d.from_numpy(q0))))
    return out, d


def main():
    sys.path.insert(0, "/root/reference/pkg/src")
    global laze
    import laze  # the real reference; only available in the build container
    only_ms = "--ms-only" in sys.argv           # regenerate only the multi-species vectors
    for name, dim, order, n, bc, opname, kw, state in ([] if only_ms else CASES):
        eager = laze.ArrayContext(mode="eager")
        probe = make_dcoll(eager, dim, order, n, bc)
        q0 = random_state(dim, probe.nelements, probe.Np, seed=11) if state == "random" else smooth_state(probe.nodes())
        res_e, d = run(eager, dim, order, n, bc, opname, kw, q0)
        res_l, _ = run(laze.ArrayContext(mode="lazy"), dim, order, n, bc, opname, kw, q0)
        payload = {"q0": q0, "vmap_m": d.vmap_m_host, "vmap_p": d.vmap_p_host, "bc_kind": d.bc_kind_host}
        for k, v in res_e.items():
            payload[f"eager_{k}"] = v
            payload[f"lazy_{k}"] = res_l[k]
            scale = max(np.abs(v).max(), 1.0)
            print(f"{name:26s} {k:5s} lazy-vs-eager rel diff {np.abs(res_l[k] - v).max() / scale:.2e}")
        np.savez_compressed(os.path.join(HERE, name + ".npz"), **payload)

    # the multi-species reactive operator (BASELINE configs[4]) through both reference contexts
    from paper_2512_17101_b200 import Mixture, MultispeciesOperator
    from tests.common import MS_GOLDEN_CASES, MS_MIXTURES, ms_state
    for name, dim, order, n, bc, ns in MS_GOLDEN_CASES:
        res = {}
        for mode in ("eager", "lazy"):
            actx = laze.ArrayContext(mode=mode)
            d = make_dcoll(actx, dim, order, n, bc)
            op = MultispeciesOperator(d, Mixture(**MS_MIXTURES[ns]))
            q0 = ms_state(op, d.nodes())
            res[mode] = np.asarray(actx.to_numpy(op.rhs(d.from_numpy(q0)).data))
        print(f"{name:26s} rhs   lazy-vs-eager rel diff {np.abs(res['lazy'] - res['eager']).max() / max(np.abs(res['eager']).max(), 1.0):.2e}")
        np.savez_compressed(os.path.join(HERE, name + ".npz"), q0=q0, eager_rhs=res["eager"], lazy_rhs=res["lazy"])

    if only_ms:
        return
    # 20 RK4 steps of the 2D isentropic-vortex-sized Euler case through the reference's eager context
    eager = laze.ArrayContext(mode="eager")
    d = make_dcoll(eager, 2, 3, 4, "periodic")
    op = EulerOperator(d)
    q0 = smooth_state(d.nodes())
    q = d.from_numpy(q0)
    t, dt = 0.0, 2e-3
    for _ in range(20):
        q = rk4_step(op.rhs, q, t, dt)
        t += dt
    np.savez_compressed(os.path.join(HERE, "euler2d_p3_rk4_20steps.npz"), q0=q0, q=np.asarray(eager.to_numpy(q.data)), dt=dt)

    # array-op level known answers restated from the reference's own tests
    actx = laze.ArrayContext(mode="lazy")
    v = actx.from_numpy(np.array([10.0, 11.0, 12.0, 13.0, 14.0]))
    sel = actx.from_numpy(np.array([4, 0, 2], dtype=np.int64))
    gather = actx.freeze(v[sel])                     # /root/reference/pkg/tests/test_scalar_ir.py:160-170
    a = np.arange(12.0).reshape(3, 4)
    b = np.arange(20.0).reshape(4, 5)
    la, lb = actx.from_numpy(a), actx.from_numpy(b)
    comp = actx.freeze(actx.np.einsum("ij,jk->ik", la, lb).reshape(5, 3)[1:4])   # test_frontend.py:126-134
    np.savez_compressed(os.path.join(HERE, "array_ops.npz"), gather=gather, einsum_reshape_slice=comp, a=a, b=b)
    print("golden vectors written to", HERE)


if __name__ == "__main__":
    main()
