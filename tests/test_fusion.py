"""Pointwise fusion (second half): chains of elementwise array operations run as ONE
`dgb_ew_program` launch -- the hand-written counterpart of the reference's fuse_loops + contract_arrays
(/root/reference/pkg/src/laze/ir_passes.py:189-284).  Results must be bit-identical to the op-by-op
kernels and to the CPU oracle, and the launch count of an un-outlined RK4 step must drop >= 4x."""
import numpy as np
import pytest

from oracle.laze_port import NumpyArrayContext
from tests.common import FARFIELD, make_dcoll, random_state

pytestmark = pytest.mark.gpu


def _ctxs():
    from paper_2512_17101_b200 import B200ArrayContext
    return B200ArrayContext(fuse_elementwise=True), B200ArrayContext(fuse_elementwise=False), NumpyArrayContext()


def _programs(actx_np):
    """Array programs in array-context arithmetic; each returns a dict of results."""
    def mixed(x, y, k, b):
        t = (x * y + 2.5) / (abs(y) + 1.0)                 # f64 chain with literals
        u = actx_np.sqrt(t * t + 1e-3) ** 1.5 - actx_np.exp(-x) + actx_np.log(abs(x) + 2.0)
        m = actx_np.maximum(x, y) - actx_np.minimum(x, 0.25)
        c = actx_np.where(x > y, u, -u) + actx_np.where(b, 1.0, m)      # comparisons feed where
        i = (k * 3 - 7) // 2 + k % 5 + (-k)                # integer arithmetic (floor semantics)
        j = i * 2 + (k > 3)                                # bool promoted to int
        f = k / 4 + i                                      # int true-division -> f64
        return {"t": t, "c": c, "i": i, "j": j, "f": f, "lt": x < 0.0, "ne": actx_np.not_equal(k, i), "eq": actx_np.equal(k % 2, 0)}

    def broadcast(x, row, col, s):
        a = x * row + col                                  # (n, m) * (m,) + (n, 1)
        return {"a": a, "b": (a - s) * (row * 2.0), "sum": actx_np.sum(a * a, axis=1)}

    def long_chain(x):
        acc = x
        for n in range(1, 70):                             # longer than one interpreter program
            acc = acc * 0.99 + (x if n % 3 else -x) * (1.0 / n)
        return {"acc": acc}

    return mixed, broadcast, long_chain


def test_fused_elementwise_bit_identical():
    fused, plain, cpu = _ctxs()
    rng = np.random.default_rng(7)
    x, y = rng.standard_normal((2, 37, 11))
    k = rng.integers(-9, 10, (37, 11))
    b = rng.random((37, 11)) > 0.5
    row, col, s = rng.standard_normal(11), rng.standard_normal((37, 1)), np.float64(0.75)
    outs = []
    for actx in (fused, plain, cpu):
        mixed, broadcast, long_chain = _programs(actx.np)
        up = actx.from_numpy
        res = {}
        res.update(mixed(up(x), up(y), up(k), up(b)))
        res.update(broadcast(up(x), up(row), up(col), float(s)))
        res.update(long_chain(up(x)))
        outs.append({name: np.asarray(actx.to_numpy(v)) for name, v in res.items()})
    f, p, c = outs
    for name in f:
        assert f[name].dtype == p[name].dtype == c[name].dtype, name
        assert np.array_equal(f[name], p[name], equal_nan=True), name        # fused == op by op, bit for bit
        if name in ("acc", "sum"):                          # exp/log/pow of libdevice vs libm differ in the last ulp
            assert np.allclose(f[name], c[name], rtol=1e-13, atol=0), name
        elif f[name].dtype != np.float64:
            assert np.array_equal(f[name], c[name]), name
        else:
            assert np.allclose(f[name], c[name], rtol=1e-13, atol=1e-15), name
    assert fused.fused_programs > 0 and fused.fused_ops > 3 * fused.fused_programs
    assert fused.launch_count * 3 < plain.launch_count


def test_rk4_step_one_pass_per_chain():
    """rk4_step written in array arithmetic (un-outlined RHS arithmetic aside): the four stage updates and
    the final combination are one launch each instead of 2 + 2 + 2 + 7."""
    from paper_2512_17101_b200 import B200ArrayContext
    from paper_2512_17101_b200.operators import NavierStokesOperator, rk4_step
    counts, results = {}, {}
    for fuse in (True, False):
        actx = B200ArrayContext(fuse_elementwise=fuse)
        d = make_dcoll(actx, 3, 3, 3, "periodic")
        op = NavierStokesOperator(d, mu=1e-2)
        q = d.from_numpy(random_state(3, d.nelements, d.Np, seed=2))
        rk4_step(op.rhs, q, 0.0, 1e-3)                      # warm-up: discretisation handle, caches
        actx.synchronize()
        n0 = actx.launch_count
        qn = rk4_step(op.rhs, q, 0.0, 1e-3)
        results[fuse] = d.to_numpy(qn)
        counts[fuse] = actx.launch_count - n0
    assert np.array_equal(results[True], results[False])
    rhs_launches = 8                                        # 4 x (dg_ns_flux + dg_ns_div)
    # 13 array operations in 4 chains (each stage state is consumed by a right-hand side, so 4 is the floor)
    assert counts[False] - rhs_launches == 13
    assert counts[True] - rhs_launches == 4


def test_generic_operator_program_fused():
    """The whole operator program with fused dispatch switched off (op by op on the generic kernels):
    elementwise chains between einsums / gathers are fused; same bits as unfused, fewer launches."""
    from paper_2512_17101_b200 import B200ArrayContext
    from paper_2512_17101_b200.operators import EulerOperator, NavierStokesOperator
    outs, launches = {}, {}
    for fuse in (True, False):
        actx = B200ArrayContext(fuse_elementwise=fuse)
        actx._fused = {}
        d = make_dcoll(actx, 3, 2, 3, "mixed")
        q0 = random_state(3, d.nelements, d.Np, seed=3)
        res = []
        for Op, kw in [(EulerOperator, {}), (NavierStokesOperator, {"mu": 2e-2})]:
            op = Op(d, farfield=FARFIELD[3], **kw)
            op.rhs(d.from_numpy(q0))
            actx.synchronize()
            n0 = actx.launch_count
            res.append(d.to_numpy(op.rhs(d.from_numpy(q0))))
            launches[(fuse, Op.__name__)] = actx.launch_count - n0
        outs[fuse] = res
    for a, b in zip(outs[True], outs[False]):
        assert np.array_equal(a, b)
    for name in ("EulerOperator", "NavierStokesOperator"):
        assert launches[(True, name)] * 2 <= launches[(False, name)], launches


def test_large_reduction_segmented():
    """actx.np.sum over 2e7 values (a norm / conservation check at production size) uses the segmented
    fixed-order reduction: deterministic, within 1e-13 of the NumPy sum, and not one thread for everything."""
    import time
    from paper_2512_17101_b200 import B200ArrayContext
    actx = B200ArrayContext()
    rng = np.random.default_rng(0)
    h = rng.standard_normal((5, 4000, 1000))
    a = actx.from_numpy(h)
    actx.to_numpy(actx.np.sum(a))
    t0 = time.time()
    s1 = float(actx.to_numpy(actx.np.sum(a * a)))
    dt = time.time() - t0
    s2 = float(actx.to_numpy(actx.np.sum(a * a)))
    assert s1 == s2
    assert abs(s1 - float((h * h).sum())) <= 1e-13 * s1
    per = actx.to_numpy(actx.np.sum(a, axis=(1, 2)))
    assert np.allclose(per, h.sum(axis=(1, 2)), rtol=0, atol=1e-9)
    assert dt < 2.0, dt
