"""``B200ArrayContext``: the reference's array-context surface executed on a B200.

Mirrors ``laze.ArrayContext`` (/root/reference/pkg/src/laze/frontend.py:309-519): same
constructor, ``from_numpy / to_numpy / freeze / compile / outline / send / receive`` and the same
``actx.np`` namespace (:257-302) and array operators (:196-250), with the same error classes
(``errors.py``).  Differences, all deliberate:

* arrays are ``DeviceArray`` handles on HBM; every op enqueues hand-written sm_100a kernels from
  ``libdgb200.so`` on the context's CUDA stream (no tracing compiler: CUDA streams instead of a
  lazy graph, so ``mode`` is always ``"eager"`` in the reference's sense);
* ``outline(f)`` dispatches BY NAME to a fused kernel when ``f.__name__`` is one of the DG
  functions of ``operators.py`` -- the reference's own call boundary
  (adfg.py:722-803; arguments/results materialised, graph_passes.py:679-681,706-707);
* only f64 / i64 / bool elements (the reference also has f32);
* torch is used for device memory, streams and ``torch.distributed`` only -- no torch math.
"""
from __future__ import annotations

import ctypes as C
import inspect
import math
from typing import Callable, Sequence

import numpy as np

from . import _cabi, errors

F64, I64, BOOL = 0, 1, 2
_NP_OF = {F64: np.dtype(np.float64), I64: np.dtype(np.int64), BOOL: np.dtype(np.bool_)}
_COMPARISONS = ("lt", "le", "gt", "ge", "eq", "ne")
_HOST_SHADOW_MAX = 1 << 16     # small from_numpy arrays keep a host copy (matrices, parameters)


def _code_of_numpy(dt) -> int:
    dt = np.dtype(dt)
    for code, ndt in _NP_OF.items():
        if ndt == dt:
            return code
    raise errors.DTypeMismatch(f"unsupported element type: {dt}")


def _torch():
    import torch
    return torch


def _torch_dtype(code: int):
    torch = _torch()
    return {F64: torch.float64, I64: torch.int64, BOOL: torch.bool}[code]


def _code_of_torch(dt) -> int:
    torch = _torch()
    return {torch.float64: F64, torch.int64: I64, torch.bool: BOOL}[dt]


def broadcast_shapes(shapes):
    """Trailing-aligned broadcast (adfg.py:114-131)."""
    rank = max((len(s) for s in shapes), default=0)
    out = []
    for k in range(rank):
        extent = 1
        for s in shapes:
            pos = len(s) - rank + k
            if pos < 0:
                continue
            e = s[pos]
            if extent == 1:
                extent = e
            elif e not in (1, extent):
                raise errors.ShapeMismatch(f"shapes {list(shapes)} are not broadcast-compatible")
        out.append(extent)
    return tuple(out)


class DeviceArray:
    """A dense or strided view of HBM owned by a ``B200ArrayContext``.  Immutable by convention:
    every operation returns a fresh array (adfg.py:291 immutability, backend.py:86 fresh outputs)."""

    __array_priority__ = 2000

    def __init__(self, actx: "B200ArrayContext", tensor, host=None):
        self.actx = actx
        self.t = tensor
        self._host = host

    # {{{ structure
    @property
    def shape(self):
        return tuple(self.t.shape)

    @property
    def dtype_code(self) -> int:
        return _code_of_torch(self.t.dtype)

    @property
    def dtype(self):
        return _NP_OF[self.dtype_code]

    @property
    def ptr(self) -> int:
        return self.t.data_ptr()

    @property
    def size(self) -> int:
        return self.t.numel()

    def __repr__(self):
        return f"DeviceArray(shape={self.shape}, dtype={self.dtype})"

    def __len__(self):
        if not self.shape:
            raise TypeError("len() of a rank-0 array")
        return self.shape[0]

    def tagged(self, axis, key, value):
        return self                      # axis tags carry no meaning for hand-fused kernels

    def reshape(self, *shape):
        if len(shape) == 1 and isinstance(shape[0], (tuple, list)):
            shape = tuple(shape[0])
        return self.actx.np.reshape(self, shape)

    def host_value(self) -> np.ndarray:
        """Host copy (cached for small arrays created by ``from_numpy``)."""
        if self._host is not None:
            return self._host
        return self.actx.to_numpy(self)
    # }}}

    # {{{ operators (frontend.py:196-218)
    def _bin(self, other, op, reflected=False):
        lhs, rhs = (other, self) if reflected else (self, other)
        return self.actx._binary_op(op, lhs, rhs)

    def __add__(self, o): return self._bin(o, "add")
    def __radd__(self, o): return self._bin(o, "add", True)
    def __sub__(self, o): return self._bin(o, "sub")
    def __rsub__(self, o): return self._bin(o, "sub", True)
    def __mul__(self, o): return self._bin(o, "mul")
    def __rmul__(self, o): return self._bin(o, "mul", True)
    def __truediv__(self, o): return self._bin(o, "truediv")
    def __rtruediv__(self, o): return self._bin(o, "truediv", True)
    def __pow__(self, o): return self._bin(o, "pow")
    def __rpow__(self, o): return self._bin(o, "pow", True)
    def __mod__(self, o): return self._bin(o, "mod")
    def __floordiv__(self, o): return self._bin(o, "floordiv")
    def __lt__(self, o): return self._bin(o, "lt")
    def __le__(self, o): return self._bin(o, "le")
    def __gt__(self, o): return self._bin(o, "gt")
    def __ge__(self, o): return self._bin(o, "ge")
    def __neg__(self): return self.actx._unary_op("neg", self)
    def __abs__(self): return self.actx._unary_op("abs", self)
    __hash__ = object.__hash__
    # }}}

    def __getitem__(self, selection):
        """ints, positive-step slices and at most one int64 index array
        (frontend.py:222-250; adfg.py:521-541)."""
        if not isinstance(selection, tuple):
            selection = (selection,)
        shape = self.shape
        if len(selection) > len(shape):
            raise errors.BadSubscript(f"{len(selection)} subscripts for rank {len(shape)}")
        selection = selection + (slice(None),) * (len(shape) - len(selection))
        basic = []
        gather = None
        for axis, sel in enumerate(selection):
            if isinstance(sel, (int, np.integer)) and not isinstance(sel, (bool, np.bool_)):
                sel = int(sel)
                if sel < 0:
                    sel += shape[axis]
                if not 0 <= sel < shape[axis]:
                    raise errors.OutOfBoundsIndex(f"index {sel} on axis {axis} leaves [0, {shape[axis]})")
                basic.append(sel)
            elif isinstance(sel, slice):
                start, stop, step = sel.indices(shape[axis])
                if step < 1:
                    raise errors.BadSubscript("only positive slice steps are supported")
                basic.append(slice(start, max(start, stop), step))
            elif isinstance(sel, DeviceArray):
                if gather is not None:
                    raise errors.BadSubscript("at most one index array per subscript")
                if sel.dtype_code != I64:
                    raise errors.DTypeMismatch("index arrays must be i64")
                gather = (axis, sel)
                basic.append(slice(None))
            else:
                raise errors.BadSubscript(f"unsupported subscript: {sel!r}")
        view = DeviceArray(self.actx, self.t[tuple(basic)])
        if gather is None:
            return view
        axis, idx = gather
        # axis position after the integer subscripts dropped their axes
        axis -= sum(1 for s in basic[:axis] if isinstance(s, int))
        return self.actx._take(view, axis, idx)


class DeferredArray(DeviceArray):
    """Result of an elementwise operation that has not been evaluated yet.

    With ``actx.fuse_elementwise`` on, ``_binary_op / _unary_op / _where`` return one of these instead of
    launching a kernel; a chain of them is evaluated by ONE ``dgb_ew_program`` launch when the value is
    first needed by anything that is not elementwise (``.t`` / ``.ptr``: a fused DG kernel, an einsum, a
    gather, a copy to the host, a graph output).  This is the hand-written counterpart of the reference's
    ``fuse_loops`` + ``contract_arrays`` (ir_passes.py:189-284) for pointwise chains: the intermediate
    arrays of the chain never exist.  Shape and element type are known without evaluating."""

    _next_seq = 0

    def __init__(self, actx, shape, code, kind, op, args, fcomp=False):
        self.actx = actx
        self._shape = tuple(int(e) for e in shape)
        self._code = code
        self._kind, self._op, self._args, self._fcomp = kind, op, args, fcomp
        self._t = None
        self._host = None
        self._seq = DeferredArray._next_seq
        DeferredArray._next_seq += 1
        # upper bound of the chain below this node (shared nodes counted once per use): long chains are cut
        # here, at creation, so that a program always fits the interpreter and evaluation never recurses deeply
        self._n = 1 + sum(a._n for a in args if isinstance(a, DeferredArray) and a.pending)
        while self._n > 48:
            big = max((a for a in args if isinstance(a, DeferredArray) and a.pending), key=lambda a: a._n)
            actx._materialize(big)
            self._n = 1 + sum(a._n for a in args if isinstance(a, DeferredArray) and a.pending)

    @property
    def t(self):
        if self._t is None:
            self.actx._materialize(self)
        return self._t

    @property
    def pending(self) -> bool:
        return self._t is None

    @property
    def shape(self):
        return self._shape

    @property
    def dtype_code(self) -> int:
        return self._code

    @property
    def size(self) -> int:
        return math.prod(self._shape)


class _OpNamespace:
    """``actx.np`` (frontend.py:257-302)."""

    def __init__(self, actx):
        self._actx = actx

    def add(self, a, b): return self._actx._binary_op("add", a, b)
    def subtract(self, a, b): return self._actx._binary_op("sub", a, b)
    def multiply(self, a, b): return self._actx._binary_op("mul", a, b)
    def divide(self, a, b): return self._actx._binary_op("truediv", a, b)
    def power(self, a, b): return self._actx._binary_op("pow", a, b)
    def maximum(self, a, b): return self._actx._binary_op("max", a, b)
    def minimum(self, a, b): return self._actx._binary_op("min", a, b)
    def greater(self, a, b): return self._actx._binary_op("gt", a, b)
    def greater_equal(self, a, b): return self._actx._binary_op("ge", a, b)
    def less(self, a, b): return self._actx._binary_op("lt", a, b)
    def less_equal(self, a, b): return self._actx._binary_op("le", a, b)
    def equal(self, a, b): return self._actx._binary_op("eq", a, b)
    def not_equal(self, a, b): return self._actx._binary_op("ne", a, b)
    def negative(self, a): return self._actx._unary_op("neg", a)
    def abs(self, a): return self._actx._unary_op("abs", a)
    def sqrt(self, a): return self._actx._unary_op("sqrt", a)
    def exp(self, a): return self._actx._unary_op("exp", a)
    def log(self, a): return self._actx._unary_op("log", a)
    def where(self, cond, a, b): return self._actx._where(cond, a, b)
    def reshape(self, a, newshape): return self._actx._reshape(a, newshape)
    def concatenate(self, arrays, axis=0): return self._actx._concatenate(arrays, axis)
    def stack(self, arrays, axis=0): return self._actx._stack(arrays, axis)
    def einsum(self, subscripts, *args): return self._actx._einsum(subscripts, args)
    def sum(self, a, axis=None): return self._actx._sum(a, axis)


class B200ArrayContext:
    """Array context whose arrays live in B200 HBM and whose ops are sm_100a kernels."""

    mode = "eager"

    def __init__(self, device: int | None = None, stream=None, comm=None, fuse_elementwise: bool = True):
        torch = _torch()
        self.fuse_elementwise = fuse_elementwise       # chains of elementwise ops -> one dgb_ew_program launch
        self.lib = _cabi.load()                       # raises ExtensionMissing: no CPU fallback
        if not torch.cuda.is_available():
            raise errors.ExtensionMissing("B200ArrayContext needs a CUDA device; there is no CPU fallback")
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        torch.cuda.set_device(self.device)
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        self.np = _OpNamespace(self)
        self.comm = comm                               # optional paper_2512_17101_b200.halo.Communicator
        self.launch_count = 0                          # kernels launched through this context
        self._scalars: dict = {}
        self._pending_sends: list = []
        self._pending_recvs: list = []
        self._discs: dict = {}
        self._keepalive: list = []
        self._pinned: list = []
        from .fused import FUSED
        self._fused = FUSED

    # {{{ plumbing
    @property
    def _st(self):
        return C.c_void_p(self.stream.cuda_stream)

    def empty(self, shape, code=F64) -> DeviceArray:
        torch = _torch()
        with torch.cuda.stream(self.stream):
            t = torch.empty(tuple(int(s) for s in shape), dtype=_torch_dtype(code), device=self.device)
        return DeviceArray(self, t)

    def synchronize(self):
        if self._pending_sends or self._pending_recvs:
            self.flush_communication()
        _cabi.check(self.lib.dgb_stream_sync(self._st), "synchronize")
        if getattr(self, "_err", None) is not None and getattr(self, "_err_armed", False):
            self._err_armed = False
            self.check_deferred_errors()      # gathers inside replayed graphs report here (to_numpy / freeze call this)

    def pinned_empty(self, shape, dtype=np.float64) -> np.ndarray:
        """Page-locked host staging buffer as a NumPy array (async H2D / D2H copies)."""
        torch = _torch()
        t = torch.empty(tuple(int(s) for s in shape), dtype=_torch_dtype(_code_of_numpy(dtype)), pin_memory=True)
        arr = t.numpy()
        self._pinned.append((arr.ctypes.data, arr.ctypes.data + max(arr.nbytes, 1), t))
        return arr

    def _is_pinned(self, arr: np.ndarray) -> bool:
        p = arr.ctypes.data
        return any(lo <= p < hi for lo, hi, _ in self._pinned)
    # }}}

    # {{{ creation / transfer (frontend.py:327-343)
    def from_numpy(self, value, pinned_staging=None) -> DeviceArray:
        value = np.asarray(value)
        code = _code_of_numpy(value.dtype)            # rejects unsupported dtypes early (:329)
        host = np.ascontiguousarray(value)
        out = self.empty(host.shape, code)
        if host.size:
            _cabi.check(self.lib.dgb_memcpy_h2d(C.c_void_p(out.ptr), C.c_void_p(host.ctypes.data),
                                                host.nbytes, self._st), "from_numpy")
            if not self._is_pinned(host):
                self.synchronize()                     # pageable source: copy must finish before `host` dies
        if host.size <= _HOST_SHADOW_MAX:
            shadow = host.copy()
            shadow.setflags(write=False)
            out._host = shadow
        return out

    # -- asynchronous upload on a second stream, so that the H2D copy of the next batch overlaps the
    #    compute + D2H of the current one (PCIe is full duplex) --------------------------------------
    @property
    def copy_stream(self):
        if getattr(self, "_copy_stream", None) is None:
            self._copy_stream = _torch().cuda.Stream(device=self.device)
        return self._copy_stream

    def from_numpy_async(self, value, after=None, out: DeviceArray | None = None) -> DeviceArray:
        """Upload a PINNED host array on the copy stream.  ``after``: an event the copy must wait for
        (e.g. the last kernel that read a buffer being recycled).  ``out``: an existing device array of
        the same shape to upload into (a streaming caller ping-pongs two of them instead of allocating
        per step; pass ``after`` = the event recorded after its last reader).  The result carries
        ``.ready``; call ``actx.wait_for(arr)`` before using it on the compute stream."""
        torch = _torch()
        host = np.ascontiguousarray(value)
        if not self._is_pinned(host):
            raise errors.LazeError("from_numpy_async needs a page-locked buffer (actx.pinned_empty)")
        cs = self.copy_stream
        if out is None:
            with torch.cuda.stream(cs):
                t = torch.empty(host.shape, dtype=_torch_dtype(_code_of_numpy(host.dtype)), device=self.device)
            out = DeviceArray(self, t)
        else:
            if tuple(out.shape) != tuple(host.shape) or out.dtype_code != _code_of_numpy(host.dtype):
                raise errors.ShapeMismatch("from_numpy_async: `out` does not match the host array")
            t = out.t
        if after is not None:
            cs.wait_event(after)
        _cabi.check(self.lib.dgb_memcpy_h2d(C.c_void_p(out.ptr), C.c_void_p(host.ctypes.data), host.nbytes,
                                            C.c_void_p(cs.cuda_stream)), "from_numpy_async")
        out.ready = torch.cuda.Event()
        out.ready.record(cs)
        t.record_stream(self.stream)
        return out

    def wait_for(self, arr: DeviceArray) -> DeviceArray:
        ev = getattr(arr, "ready", None)
        if ev is not None:
            self.stream.wait_event(ev)
        return arr

    @property
    def d2h_stream(self):
        if getattr(self, "_d2h_stream", None) is None:
            self._d2h_stream = _torch().cuda.Stream(device=self.device)
        return self._d2h_stream

    def to_numpy_async(self, value: DeviceArray, out: np.ndarray):
        """D2H into a pinned buffer on a dedicated download stream, ordered after everything enqueued
        so far on the compute stream; does not block the host or later kernels.  Returns the event
        that marks the copy done (``stream.wait_event(ev)`` / ``ev.synchronize()`` before reading)."""
        torch = _torch()
        src = self._contiguous(value)
        done = torch.cuda.Event()
        done.record(self.stream)
        ds = self.d2h_stream
        ds.wait_event(done)
        _cabi.check(self.lib.dgb_memcpy_d2h(C.c_void_p(out.ctypes.data), C.c_void_p(src.ptr), out.nbytes,
                                            C.c_void_p(ds.cuda_stream)), "to_numpy_async")
        ev = torch.cuda.Event()
        ev.record(ds)
        src.t.record_stream(ds)
        self._keepalive = [src]
        return ev

    def to_numpy(self, value, out=None) -> np.ndarray:
        if not isinstance(value, DeviceArray):
            return np.asarray(value)
        src = self._contiguous(value)
        host = out if out is not None else np.empty(src.shape, dtype=_NP_OF[src.dtype_code])
        if src.size:
            _cabi.check(self.lib.dgb_memcpy_d2h(C.c_void_p(host.ctypes.data), C.c_void_p(src.ptr),
                                                host.nbytes, self._st), "to_numpy")
        self.synchronize()
        return host

    def freeze(self, what):
        """Arrays are already evaluated; ``freeze`` returns host values like the reference's
        (frontend.py:526-552)."""
        if isinstance(what, dict):
            return {k: self.to_numpy(v) for k, v in what.items()}
        return self.to_numpy(what)

    def placeholder(self, name, shape, dtype=None):
        raise errors.LazeError("eager contexts have no placeholders")     # frontend.py:336-337
    # }}}

    # {{{ operands
    def _scalar(self, value, code) -> DeviceArray:
        """Rank-0 device array holding a literal.  Outside a graph capture the arrays are cached (LRU,
        4096 entries).  Inside a capture the cache is neither read nor written: the array is created by a
        captured fill kernel in the graph's own memory pool, so a graph never holds the address of a
        cache entry that a later eviction could free, and nothing synchronises the capturing stream."""
        torch = _torch()
        if getattr(self, "_capturing", False):
            with torch.cuda.stream(self.stream):
                t = torch.full((), float(value) if code == F64 else (bool(value) if code == BOOL else int(value)),
                               dtype=_torch_dtype(code), device=self.device)
            self.launch_count += 1
            return DeviceArray(self, t)
        key = (code, float(value) if code == F64 else int(value))
        arr = self._scalars.pop(key, None)
        if arr is None:
            while len(self._scalars) >= 4096:
                self._scalars.pop(next(iter(self._scalars)))      # least recently used first
            arr = self.from_numpy(np.asarray(value, dtype=_NP_OF[code]))
        self._scalars[key] = arr                                   # (re)insert as most recently used
        return arr

    def _as_operand(self, value):
        """-> (DeviceArray | None, (python scalar, weak dtype code) | None)   (frontend.py:349-362)"""
        if isinstance(value, DeviceArray):
            return value, None
        if isinstance(value, (bool, np.bool_)):
            return None, (bool(value), BOOL)
        if isinstance(value, (int, np.integer)):
            return None, (int(value), I64)
        if isinstance(value, (float, np.floating)):
            return None, (float(value), F64)
        if isinstance(value, np.ndarray):
            if value.ndim == 0:
                return self._as_operand(value[()])
            return self.from_numpy(value), None
        if hasattr(value, "data") and isinstance(getattr(value, "data"), DeviceArray):
            return value.data, None                    # DOFArray
        raise errors.LazeError(f"cannot use {type(value).__name__} as an operand")

    @staticmethod
    def _combine(a, b):
        """dtype of a binary combination with weak literals (adfg.py:885-898)."""
        (ta, wa), (tb, wb) = a, b
        rank = {BOOL: 0, I64: 1, F64: 3}
        if wa == wb:
            return (ta if rank[ta] >= rank[tb] else tb), wa
        strong, weak = (tb, ta) if wa else (ta, tb)
        if weak == F64 and strong in (I64, BOOL):
            return F64, False
        if weak == I64 and strong == BOOL:
            return I64, False
        return strong, False

    def _materialize_operands(self, values):
        ops = [self._as_operand(v) for v in values]
        if all(node is None for node, _ in ops):
            raise errors.LazeError("at least one operand must be an array")
        return ops
    # }}}

    # {{{ fused elementwise programs (ir_passes.py:189-284: fuse_loops + contract_arrays, for pointwise chains)
    class _Literal:
        """A literal operand of a deferred elementwise operation: an immediate of the program."""
        __slots__ = ("value", "dtype_code")
        shape = ()

        def __init__(self, value, code):
            self.value, self.dtype_code = value, code

    def _literal(self, value, code):
        if self.fuse_elementwise:
            return B200ArrayContext._Literal(value, code)
        return self._scalar(value, code)

    def _pending_dag(self, root):
        """Pending nodes reachable from ``root`` in issue order, and the number of references each gets
        from inside that set."""
        seen, stack, inner = {}, [root], {}
        while stack:
            x = stack.pop()
            if id(x) in seen:
                continue
            seen[id(x)] = x
            for a in x._args:
                if isinstance(a, DeferredArray) and a.pending:
                    inner[id(a)] = inner.get(id(a), 0) + 1
                    stack.append(a)
        return sorted(seen.values(), key=lambda n: n._seq), inner

    def _materialize(self, root: "DeferredArray"):
        """Evaluate ``root`` (and every pending node below it) with ONE interpreter launch; pending nodes
        of the same shape that something else still refers to are written out by the same launch."""
        import struct
        import sys
        while True:
            order, inner = self._pending_dag(root)
            # leaves, immediates, instructions
            leaves, leaf_of, consts, const_of = [], {}, [], {}
            prog = []                          # (kind, op, node-or-None, [operand keys], fcomp)
            val_dtype = {}

            def key_of(a):
                if isinstance(a, B200ArrayContext._Literal):
                    bits = (struct.unpack("<Q", struct.pack("<d", float(a.value)))[0] if a.dtype_code == F64
                            else (int(bool(a.value)) if a.dtype_code == BOOL else int(a.value) & 0xFFFFFFFFFFFFFFFF))
                    k = ("c", bits, a.dtype_code)
                    if k not in const_of:
                        const_of[k] = len(consts)
                        consts.append(bits)
                        prog.append((_cabi.EW_CONST, 0, k, [const_of[k]], False))
                        val_dtype[k] = a.dtype_code
                    return k
                if isinstance(a, DeferredArray) and a.pending:
                    return ("n", id(a))
                k = ("l", id(a))
                if k not in leaf_of:
                    leaf_of[k] = len(leaves)
                    leaves.append(a)
                    prog.append((_cabi.EW_LOAD, 0, k, [leaf_of[k]], False))
                    val_dtype[k] = a.dtype_code
                return k

            for node in order:
                ops = [key_of(a) for a in node._args]
                k = ("n", id(node))
                prog.append((node._kind, node._op, k, ops, node._fcomp))
                val_dtype[k] = node._code
            # extra outputs: pending nodes of root's shape that are referenced from outside this DAG
            outs = [root]
            for node in order:
                if node is root or node._shape != root._shape or len(outs) >= _cabi.EW_MAX_OUTS:
                    continue
                if sys.getrefcount(node) - 3 - inner.get(id(node), 0) > 0:     # `order`, `node`, getrefcount's argument
                    outs.append(node)
            # registers by liveness (values die after their last use; outputs live to the end)
            last = {}
            for i, (_, _, k, ops, _) in enumerate(prog):
                if prog[i][0] not in (_cabi.EW_LOAD, _cabi.EW_CONST):
                    for o in ops:
                        last[o] = i
            for o in outs:
                last[("n", id(o))] = len(prog)
            free, reg, ins, ok = list(range(_cabi.EW_MAX_REGS - 1, -1, -1)), {}, [], True
            for i, (kind, op, k, ops, fcomp) in enumerate(prog):
                srcs = [] if kind in (_cabi.EW_LOAD, _cabi.EW_CONST) else ops
                for o in set(srcs):
                    if last.get(o) == i:
                        free.append(reg[o])            # the destination may reuse a dying source register
                if k not in last:
                    last[k] = i                        # value never used (cannot happen for DAG nodes)
                if not free:
                    ok = False
                    break
                reg[k] = free.pop()
                if kind in (_cabi.EW_LOAD, _cabi.EW_CONST):
                    ins.append((kind, op, reg[k], ops[0], 0, 0, 0, 0, 0, val_dtype[k], 0))
                else:
                    r = [reg[o] for o in srcs] + [0] * (3 - len(srcs))
                    dt = [val_dtype[o] for o in srcs] + [0] * (3 - len(srcs))
                    ins.append((kind, op, reg[k], r[0], r[1], r[2], dt[0], dt[1], dt[2], val_dtype[k], int(fcomp)))
            if ok and len(ins) <= _cabi.EW_MAX_INS and len(leaves) <= _cabi.EW_MAX_LEAVES and len(consts) <= _cabi.EW_MAX_CONSTS:
                break
            # too large for one program: evaluate the pending operands of the root first, then retry
            pend = [a for a in root._args if isinstance(a, DeferredArray) and a.pending]
            if not pend:
                raise errors.LazeError("elementwise program does not fit the interpreter limits")
            for a in pend:
                self._materialize(a)
        shape = root._shape
        total = math.prod(shape)
        results = [self.empty(shape, o._code) for o in outs]
        if total:
            pg = _cabi.EwProg()
            pg.nins, pg.nleaves, pg.nouts, pg.rank, pg.total = len(ins), len(leaves), len(outs), len(shape), total
            need_index = 0
            for k, e in enumerate(shape):
                pg.ext[k] = e
            for k, bits in enumerate(consts):
                pg.consts[k] = bits
            for k, lf in enumerate(leaves):
                st = self._bstrides(lf, shape)
                dense, scalar, run = True, True, 1
                for ax in range(len(shape) - 1, -1, -1):
                    if shape[ax] != 1:
                        dense = dense and st[ax] == run
                        scalar = scalar and st[ax] == 0
                    run *= shape[ax]
                mode = 1 if dense else (2 if scalar else 0)
                need_index |= int(mode == 0)
                pg.leaf[k].dev, pg.leaf[k].dtype, pg.leaf[k].mode = lf.ptr, lf.dtype_code, mode
                for ax, v in enumerate(st):
                    pg.leaf[k].stride[ax] = v
            pg.need_index = need_index
            for k, (o, res) in enumerate(zip(outs, results)):
                pg.out[k].dev, pg.out[k].dtype, pg.out[k].reg = res.ptr, o._code, reg[("n", id(o))]
            for k, f in enumerate(ins):
                (pg.ins[k].kind, pg.ins[k].op, pg.ins[k].dst, pg.ins[k].a, pg.ins[k].b, pg.ins[k].c, pg.ins[k].adt,
                 pg.ins[k].bdt, pg.ins[k].cdt, pg.ins[k].odt, pg.ins[k].fcomp) = f
            _cabi.check(self.lib.dgb_ew_program(C.byref(pg), self._st), "elementwise program")
            self.launch_count += 1
            self.fused_programs = getattr(self, "fused_programs", 0) + 1
            self.fused_ops = getattr(self, "fused_ops", 0) + len(order)
        for o, res in zip(outs, results):
            o._t = res.t
            o._args = ()                       # the chain below is no longer needed

    def materialize(self, value):
        """Force the evaluation of deferred elementwise results inside ``value`` (array, DOFArray, dict, sequence)."""
        if isinstance(value, DeferredArray):
            value.t
        elif isinstance(value, dict):
            for v in value.values():
                self.materialize(v)
        elif isinstance(value, (list, tuple)):
            for v in value:
                self.materialize(v)
        elif hasattr(value, "data") and isinstance(getattr(value, "data"), DeviceArray):
            self.materialize(value.data)
        return value
    # }}}

    # {{{ elementwise (frontend.py:374-410)
    @staticmethod
    def _bstrides(arr: DeviceArray, out_shape):
        shape, strides = arr.shape, arr.t.stride()
        off = len(out_shape) - len(shape)
        res = [0] * len(out_shape)
        for j, (e, s) in enumerate(zip(shape, strides)):
            res[off + j] = 0 if (e == 1 and out_shape[off + j] != 1) else s
        return res

    def _binary_op(self, op, a, b):
        (na, la), (nb, lb) = self._materialize_operands((a, b))
        ta = (na.dtype_code, False) if na is not None else (la[1], True)
        tb = (nb.dtype_code, False) if nb is not None else (lb[1], True)
        both, _ = self._combine(ta, tb)
        if op in _COMPARISONS:
            out_code = BOOL
        elif op == "truediv":
            out_code = F64
        else:
            out_code = both
        if na is None:
            na = self._literal(la[0], F64 if both == F64 else la[1])
        if nb is None:
            nb = self._literal(lb[0], F64 if both == F64 else lb[1])
        out_shape = broadcast_shapes([na.shape, nb.shape])
        if len(out_shape) > 8:
            raise errors.ShapeMismatch(f"rank {len(out_shape)} exceeds the maximum of 8")
        if self.fuse_elementwise:
            return DeferredArray(self, out_shape, out_code, _cabi.EW_BINARY, _cabi.BINOPS[op], [na, nb],
                                 fcomp=(na.dtype_code == F64 or nb.dtype_code == F64))
        out = self.empty(out_shape, out_code)
        sa, sb = self._bstrides(na, out_shape), self._bstrides(nb, out_shape)
        _cabi.check(self.lib.dgb_ew_binary(
            _cabi.BINOPS[op], out.ptr, out_code, na.ptr, na.dtype_code, _cabi.i64_array(sa),
            nb.ptr, nb.dtype_code, _cabi.i64_array(sb), len(out_shape), _cabi.i64_array(out_shape),
            self._st), op)
        self.launch_count += 1
        return out

    def _unary_op(self, op, a):
        node, lit = self._as_operand(a)
        if node is None:
            raise errors.LazeError("at least one operand must be an array")
        out_code = F64 if op in ("sqrt", "exp", "log") else node.dtype_code
        if self.fuse_elementwise:
            return DeferredArray(self, node.shape, out_code, _cabi.EW_UNARY, _cabi.UNOPS[op], [node])
        node = self._contiguous(node)
        out = self.empty(node.shape, out_code)
        _cabi.check(self.lib.dgb_ew_unary(_cabi.UNOPS[op], out.ptr, out_code, node.ptr, node.dtype_code,
                                          node.size, self._st), op)
        self.launch_count += 1
        return out

    def _where(self, cond, a, b):
        (nc, lc), (na, la), (nb, lb) = self._materialize_operands((cond, a, b))
        ta = (na.dtype_code, False) if na is not None else (la[1], True)
        tb = (nb.dtype_code, False) if nb is not None else (lb[1], True)
        out_code, _ = self._combine(ta, tb)
        if nc is None:
            nc = self._literal(lc[0], lc[1])
        if na is None:
            na = self._literal(la[0], F64 if out_code == F64 else la[1])
        if nb is None:
            nb = self._literal(lb[0], F64 if out_code == F64 else lb[1])
        out_shape = broadcast_shapes([nc.shape, na.shape, nb.shape])
        if self.fuse_elementwise:
            if len(out_shape) > 8:
                raise errors.ShapeMismatch(f"rank {len(out_shape)} exceeds the maximum of 8")
            return DeferredArray(self, out_shape, out_code, _cabi.EW_WHERE, 0, [na, nb, nc])
        out = self.empty(out_shape, out_code)
        _cabi.check(self.lib.dgb_ew_where(
            out.ptr, out_code, nc.ptr, nc.dtype_code, _cabi.i64_array(self._bstrides(nc, out_shape)),
            na.ptr, na.dtype_code, _cabi.i64_array(self._bstrides(na, out_shape)),
            nb.ptr, nb.dtype_code, _cabi.i64_array(self._bstrides(nb, out_shape)),
            len(out_shape), _cabi.i64_array(out_shape), self._st), "where")
        self.launch_count += 1
        return out
    # }}}

    # {{{ structural ops (frontend.py:423-463)
    def _node_of(self, value) -> DeviceArray:
        node, lit = self._as_operand(value)
        if node is None:
            node = self._scalar(lit[0], lit[1])
        return node

    def _contiguous(self, arr: DeviceArray) -> DeviceArray:
        if arr.t.is_contiguous():
            return arr
        out = self.empty(arr.shape, arr.dtype_code)
        if arr.size:
            _cabi.check(self.lib.dgb_copy_strided(out.ptr, out.dtype_code, arr.ptr, arr.dtype_code,
                                                  _cabi.i64_array(arr.t.stride()), len(arr.shape),
                                                  _cabi.i64_array(arr.shape), self._st), "copy")
            self.launch_count += 1
        return out

    def _reshape(self, a, newshape):
        node = self._node_of(a)
        newshape = _resolve_reshape(node.shape, newshape)
        if math.prod(newshape) != node.size:
            raise errors.ShapeMismatch(f"cannot reshape {node.shape} to {newshape}")
        node = self._contiguous(node)
        return DeviceArray(self, node.t.view(newshape))

    def _copy_d2d(self, dst: DeviceArray, src: DeviceArray):
        if dst.size:
            nbytes = dst.size * _NP_OF[dst.dtype_code].itemsize
            _cabi.check(self.lib.dgb_memcpy_d2d(C.c_void_p(dst.ptr), C.c_void_p(src.ptr), nbytes, self._st), "d2d")

    def _scatter_into(self, out: DeviceArray, view, src: DeviceArray):
        """Copy ``src`` into the (strided) torch view ``view`` of ``out``."""
        if not src.size:
            return
        off = (view.data_ptr() - out.t.data_ptr())
        _cabi.check(self.lib.dgb_copy_scatter(
            out.ptr + off, out.dtype_code, _cabi.i64_array(view.stride()), src.ptr, src.dtype_code,
            _cabi.i64_array(src.t.stride()), len(src.shape), _cabi.i64_array(src.shape), self._st), "copy")
        self.launch_count += 1

    def _concatenate(self, arrays, axis):
        nodes = [self._node_of(a) for a in arrays]
        if not nodes:
            raise errors.ShapeMismatch("concatenate needs at least one array")
        rank = len(nodes[0].shape)
        axis = axis % rank if rank else 0
        base = list(nodes[0].shape)
        total = 0
        code = nodes[0].dtype_code
        for n in nodes:
            s = list(n.shape)
            if len(s) != rank or s[:axis] + s[axis + 1:] != base[:axis] + base[axis + 1:]:
                raise errors.ShapeMismatch("concatenate: shapes differ off the joined axis")
            total += s[axis]
            code = self._combine((code, False), (n.dtype_code, False))[0]
        base[axis] = total
        out = self.empty(base, code)
        pos = 0
        for n in nodes:
            sl = [slice(None)] * rank
            sl[axis] = slice(pos, pos + n.shape[axis])
            self._scatter_into(out, out.t[tuple(sl)], n)
            pos += n.shape[axis]
        return out

    def _stack(self, arrays, axis):
        nodes = [self._node_of(a) for a in arrays]
        if not nodes:
            raise errors.ShapeMismatch("stack needs at least one array")
        shape = nodes[0].shape
        code = nodes[0].dtype_code
        for n in nodes:
            if n.shape != shape:
                raise errors.ShapeMismatch("stack: all arrays must have the same shape")
            code = self._combine((code, False), (n.dtype_code, False))[0]
        rank = len(shape) + 1
        axis = axis % rank
        out = self.empty(shape[:axis] + (len(nodes),) + shape[axis:], code)
        for k, n in enumerate(nodes):
            sl = [slice(None)] * rank
            sl[axis] = k
            self._scatter_into(out, out.t[tuple(sl)], n)
        return out

    def _take(self, arr: DeviceArray, axis: int, idx: DeviceArray) -> DeviceArray:
        arr = self._contiguous(arr)
        idx = self._contiguous(idx)
        shape = arr.shape
        outer = math.prod(shape[:axis])
        inner = math.prod(shape[axis + 1:])
        out = self.empty(shape[:axis] + idx.shape + shape[axis + 1:], arr.dtype_code)
        if getattr(self, "_capturing", False):
            # inside a CUDA-graph capture: no host synchronisation; a bad index raises the context's
            # device-side flag, checked after every replay (the eager warm-up run has range-checked
            # this very gather already)
            _cabi.check(self.lib.dgb_take_deferred(out.ptr, arr.ptr, arr.dtype_code, idx.ptr, outer, shape[axis], inner,
                                                   idx.size, C.c_void_p(self._err_flag().data_ptr()), self._st),
                        "index array")
        else:
            _cabi.check(self.lib.dgb_take(out.ptr, arr.ptr, arr.dtype_code, idx.ptr, outer, shape[axis], inner,
                                          idx.size, self._st), "index array")
        self.launch_count += 1
        return out

    def _err_flag(self):
        if getattr(self, "_err", None) is None:
            torch = _torch()
            with torch.cuda.stream(self.stream):
                self._err = torch.zeros(1, dtype=torch.int32, device=self.device)
        return self._err

    def check_deferred_errors(self):
        """Raise ``OutOfBoundsIndex`` if a gather inside a replayed graph left its range (synchronises)."""
        if getattr(self, "_err", None) is not None and int(self._err.item()) != 0:
            self._err.zero_()
            raise errors.OutOfBoundsIndex("index array leaves [0, extent) (detected in a captured graph)")

    def _einsum(self, subscripts, args):
        nodes = [self._node_of(a) for a in args]
        subscripts = subscripts.replace(" ", "")
        if "->" not in subscripts:
            raise errors.BadSubscript(f"einsum subscripts need an explicit '->': {subscripts!r}")
        lhs, out_sub = subscripts.split("->")
        in_subs = lhs.split(",")
        if len(in_subs) != len(nodes):
            raise errors.BadSubscript(f"{len(in_subs)} subscript groups for {len(nodes)} operands")
        if not 1 <= len(nodes) <= 3:
            raise errors.BadSubscript("einsum takes one to three operands on this context")
        extent = {}
        for sub, n in zip(in_subs, nodes):
            if (sub and not sub.isalpha()) or len(sub) != len(n.shape):
                raise errors.BadSubscript(f"subscript {sub!r} does not fit shape {n.shape}")
            for letter, e in zip(sub, n.shape):
                if extent.setdefault(letter, e) != e:
                    raise errors.ShapeMismatch(f"letter {letter!r} bound to extents {extent[letter]} and {e}")
        if len(set(out_sub)) != len(out_sub):
            raise errors.BadSubscript(f"repeated letter in output subscript: {out_sub!r}")
        for letter in out_sub:
            if letter not in extent:
                raise errors.BadSubscript(f"output letter {letter!r} does not appear in any input")
        reduced = []
        for sub in in_subs:
            for letter in sub:
                if letter not in out_sub and letter not in reduced:
                    reduced.append(letter)
        letters = list(out_sub) + reduced
        if len(letters) > 8:
            raise errors.BadSubscript("einsum uses more than 8 distinct letters")
        ops = []
        for n in nodes:
            if n.dtype_code != F64:
                f = self.empty(n.shape, F64)
                _cabi.check(self.lib.dgb_copy_strided(f.ptr, F64, n.ptr, n.dtype_code, _cabi.i64_array(n.t.stride()),
                                                      len(n.shape), _cabi.i64_array(n.shape), self._st), "cast")
                self.launch_count += 1
                n = f
            ops.append(n)
        strides = []
        for sub, n in zip(in_subs, ops):
            st = n.t.stride()
            strides += [sum(s for l2, s in zip(sub, st) if l2 == letter) for letter in letters]
        out = self.empty(tuple(extent[l] for l in out_sub), F64)
        ptrs = (C.c_void_p * 3)(*[o.ptr for o in ops] + [None] * (3 - len(ops)))
        _cabi.check(self.lib.dgb_einsum(out.ptr, len(ops), ptrs, _cabi.i64_array(strides), len(out_sub),
                                        len(letters), _cabi.i64_array([extent[l] for l in letters]), self._st),
                    "einsum")
        self.launch_count += 1
        return out

    def _sum(self, a, axis):
        node = self._node_of(a)
        rank = len(node.shape)
        if axis is None:
            red = set(range(rank))
        elif isinstance(axis, int):
            red = {axis % rank}
        else:
            red = {ax % rank for ax in axis}
        letters = "abcdefgh"[:rank]
        out = "".join(letters[k] for k in range(rank) if k not in red)
        return self._einsum(f"{letters}->{out}", (node,))
    # }}}

    # {{{ compile / outline (frontend.py:485-519, 606-679)
    def compile(self, f: Callable, graph: bool = False) -> "CompiledFunction":
        """``graph=True``: per signature, the first call runs ``f`` eagerly (validating it and warming
        every cache), the second captures it into ONE CUDA graph over static argument buffers, and
        later calls copy the arguments in and replay the graph -- the B200 counterpart of the
        reference's trace-once / execute-many ``CompiledFunction`` (frontend.py:606-679) for glue
        that is not hand-fused: same kernels, no per-op Python dispatch and no launch gaps.
        Only for functions of device arrays whose control flow does not depend on array values."""
        return CompiledFunction(self, f, graph=graph)

    def outline(self, f: Callable) -> Callable:
        """Named call boundary.  DG functions known to ``fused.FUSED`` whose body is the one the kernels
        implement (source fingerprint, ``fused.body_matches``) run as fused kernels; any other function
        runs its body op by op on the device (the reference's eager behaviour, :494-495)."""
        impl = self._fused.get(f.__name__)
        if impl is None:
            return f
        from . import fused
        if not fused.supported(f):        # e.g. a species count the fused kernels are not instantiated for
            return f
        if not fused.body_matches(f):
            # same name, different body (another EOS, another flux ...): the hand-written kernel would
            # silently compute the built-in physics.  Run the body itself, op by op, on the device.
            fused.warn_mismatch(f.__name__)
            return f
        actx = self

        def fused_call(*args):
            return impl(actx, f, *args)

        fused_call.__name__ = f.__name__
        fused_call.fused = True
        return fused_call
    # }}}

    # {{{ communication (frontend.py:469-478)
    # The reference records Send / Receive nodes and its distributed executor posts every receive of a
    # batch up front, then the sends (distpart.py:168-196).  Here ``receive`` hands out an array whose
    # transfer is posted lazily and ``send`` queues its payload; the first use of any received array (or
    # ``actx.synchronize()``) posts everything queued so far as ONE batch of point-to-point operations
    # (an NCCL group: no ordering deadlock between ranks that both receive first), on the context's stream.
    @staticmethod
    def _code_of_any(dtype) -> int:
        if dtype is None:
            return F64
        if isinstance(dtype, (int, np.integer)) and int(dtype) in _NP_OF:
            return int(dtype)
        name = getattr(dtype, "value", None)                      # the reference's DType enum (adfg.py:39-45)
        if isinstance(name, str):
            table = {"f64": F64, "i64": I64, "bool": BOOL}
            if name not in table:
                raise errors.DTypeMismatch(f"unsupported element type: {name}")
            return table[name]
        return _code_of_numpy(dtype)

    def receive(self, source: int, tag: int, shape: Sequence[int], dtype=None) -> DeviceArray:
        if self.comm is None:
            raise errors.CommunicationInSingleProcessGraph(
                f"receive (source={source}, tag={tag}) on a context without a communicator")
        return ReceivedArray(self, int(source), int(tag), tuple(int(e) for e in shape), self._code_of_any(dtype))

    def send(self, value, dest: int, tag: int, *, stapled_to):
        if self.comm is None:
            raise errors.CommunicationInSingleProcessGraph(
                f"send (dest={dest}, tag={tag}) on a context without a communicator")
        self._pending_sends.append((self._contiguous(self._node_of(value)), int(dest), int(tag)))
        return stapled_to

    def flush_communication(self):
        """Post every queued send and receive as one batch and wait for it on the context's stream."""
        sends, recvs = self._pending_sends, self._pending_recvs
        if not sends and not recvs:
            return
        self._pending_sends, self._pending_recvs = [], []
        torch = _torch()
        with torch.cuda.stream(self.stream):
            self.comm.exchange([(a.t, dest, tag) for a, dest, tag in sends],
                               [(r._buf.t, r._source, r._tag) for r in recvs])
        for r in recvs:
            r._arrived = True
    # }}}


class ReceivedArray(DeviceArray):
    """Result of ``actx.receive``: the buffer exists at once, the transfer is posted with the next batch."""

    def __init__(self, actx, source, tag, shape, code):
        self.actx = actx
        self._buf = actx.empty(shape, code)
        self._source, self._tag, self._arrived = source, tag, False
        self._host = None
        actx._pending_recvs.append(self)

    @property
    def t(self):
        if not self._arrived:
            self.actx.flush_communication()
        return self._buf.t

    @property
    def shape(self):
        return self._buf.shape

    @property
    def dtype_code(self) -> int:
        return self._buf.dtype_code

    @property
    def size(self) -> int:
        return self._buf.size


class CompiledFunction:
    """Per-signature bookkeeping like the reference's (frontend.py:606-679); nothing is traced --
    the function body runs on the stream.  ndarray arguments are uploaded and ndarray results
    returned; ``DeviceArray`` arguments stay on the device and so do the results."""

    def __init__(self, actx, f, graph: bool = False):
        self.actx, self.f = actx, f
        self.signatures: set = set()
        self.trace_count = 0
        self.execution_count = 0
        self.cache_hits = 0
        self.use_graph = graph
        self._graphs: dict = {}          # signature -> (CUDAGraph, static inputs, static outputs)
        self._seen: dict = {}            # signature -> number of eager calls so far
        self.replays = 0

    # {{{ CUDA-graph path
    def _graph_call(self, sig, call_args):
        torch = _torch()
        actx = self.actx
        names = list(call_args)
        if any(hasattr(v, "data") and not isinstance(v, DeviceArray) for v in call_args.values()):
            return None                   # containers (DOFArray ...) are not flattened here: eager
        dev = dict(call_args)
        # scalars are arguments, not baked constants (frontend.py:665-668): a graph is keyed on their values
        sig = (sig, tuple(v for v in call_args.values() if not isinstance(v, DeviceArray)))
        entry = self._graphs.get(sig)
        if entry is None:
            if self._seen.get(sig, 0) < 1:          # first call of this signature: plain eager run
                self._seen[sig] = self._seen.get(sig, 0) + 1
                return None
            static = {n: (actx.empty(v.shape, v.dtype_code) if isinstance(v, DeviceArray) else v) for n, v in dev.items()}
            for n in names:
                if isinstance(dev[n], DeviceArray):
                    actx._copy_d2d(static[n], actx._contiguous(dev[n]))
            actx.synchronize()
            g = torch.cuda.CUDAGraph()
            cap = torch.cuda.Stream(device=actx.device)
            cap.wait_stream(actx.stream)
            home, actx.stream = actx.stream, cap
            actx._capturing = True
            try:
                with torch.cuda.graph(g, stream=cap):
                    out = actx.materialize(self.f(**static))
            finally:
                actx._capturing = False
                actx.stream = home
            home.wait_stream(cap)
            entry = (g, static, out)
            self._graphs[sig] = entry
        g, static, out = entry
        for n in names:
            if isinstance(dev[n], DeviceArray):
                actx._copy_d2d(static[n], actx._contiguous(dev[n]))
        with torch.cuda.stream(actx.stream):
            g.replay()
        self.replays += 1
        if getattr(actx, "_err", None) is not None:
            actx._err_armed = True        # the next synchronisation point looks at the device-side error flag

        def fresh(a):                     # results live in the graph's pool: hand out copies
            if isinstance(a, DeviceArray):
                c = actx.empty(a.shape, a.dtype_code)
                actx._copy_d2d(c, a)
                return c
            return a
        if isinstance(out, dict):
            return {k: fresh(v) for k, v in out.items()}
        return fresh(out)
    # }}}

    def __call__(self, *args, **kwargs):
        bound = inspect.signature(self.f).bind(*args, **kwargs)
        bound.apply_defaults()
        sig = []
        on_device = False
        call_args = {}
        for name, value in bound.arguments.items():
            if value is None:
                sig.append((name, ("none",)))
            elif isinstance(value, (bool, np.bool_, int, np.integer, float, np.floating)):
                sig.append((name, ("scalar", type(value).__name__)))
            elif isinstance(value, np.ndarray):
                sig.append((name, ("array", value.shape, str(value.dtype))))
                value = self.actx.from_numpy(value)
            elif isinstance(value, DeviceArray) or hasattr(value, "data"):
                on_device = True
                sig.append((name, ("device", tuple(getattr(value, "shape", ())))))
            else:
                raise errors.SignatureUnsupported(
                    f"compiled functions take arrays, scalars, or None; got {type(value).__name__}")
            call_args[name] = value
        sig = tuple(sig)
        if sig in self.signatures:
            self.cache_hits += 1
        else:
            self.signatures.add(sig)
            self.trace_count += 1
        self.execution_count += 1
        if self.use_graph and on_device and not kwargs:
            res = self._graph_call(sig, call_args)
            if res is not None:
                return res
        out = self.f(**call_args)
        if on_device:
            return out
        if isinstance(out, dict):
            return {k: self.actx.to_numpy(v) for k, v in out.items()}
        return self.actx.to_numpy(out)


def _resolve_reshape(old_shape, newshape):
    """frontend.py:689-707."""
    if isinstance(newshape, (int, np.integer)):
        newshape = (int(newshape),)
    newshape = tuple(int(e) for e in newshape)
    if newshape.count(-1) > 1:
        raise errors.ShapeMismatch("at most one extent may be -1")
    if -1 in newshape:
        size = math.prod(old_shape)
        known = 1
        for e in newshape:
            if e != -1:
                known *= e
        if known == 0 or size % known:
            raise errors.ShapeMismatch(f"cannot infer extent: {old_shape} to {newshape}")
        newshape = tuple(size // known if e == -1 else e for e in newshape)
    return newshape
