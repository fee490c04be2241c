"""Export of a traced array program in the reference CLI's JSON program format.

``GraphExportContext`` is a third array context for the operator program (next to the B200 context and the CPU
oracle): it executes nothing, it *records*.  Running ``NavierStokesOperator(dcoll).rhs(q)`` on it yields the
dataflow graph of the right-hand side -- ``expression`` / ``einsum`` / ``index`` / ``reshape`` / ``stack`` /
``concatenate`` nodes, the outlined DG functions as ``functions`` + ``call`` nodes -- as the document
``laze oracle prog.json`` / ``laze run prog.json`` replay independently of this package:

* document layout and node kinds: /root/reference/pkg/src/laze/cli.py:160-335 (loader) and :434-576
  (``graph_to_doc``, the serializer this module is the counterpart of);
* expression text: /root/reference/pkg/src/laze/expr.py:386-426 (``to_str``) as parsed by cli.py:66-129;
* trailing-aligned broadcast loads: /root/reference/pkg/src/laze/frontend.py:364-392;
* outlined functions: parameters ``_p0, _p1, ...``, a single result named ``out`` (frontend.py:488-519, 575).

Meant for small cases (arrays are embedded as nested lists).
"""
from __future__ import annotations

import numpy as np

from . import errors

_DT = {np.dtype(np.float64): "f64", np.dtype(np.float32): "f32", np.dtype(np.int64): "i64", np.dtype(np.bool_): "bool"}
_BIN_SYMBOL = {"add": "+", "sub": "-", "mul": "*", "truediv": "/", "floordiv": "//", "mod": "%", "pow": "**",
               "lt": "<", "le": "<=", "gt": ">", "ge": ">=", "eq": "==", "ne": "!="}
_COMPARE = {"lt", "le", "gt", "ge", "eq", "ne"}


class _Scope:
    def __init__(self, prefix="_n"):
        self.nodes: dict[str, dict] = {}
        self.count = 0
        self.prefix = prefix

    def add(self, spec, name=None):
        if name is None:
            name = f"{self.prefix}{self.count}"
            self.count += 1
        if name in self.nodes:
            raise errors.LazeError(f"duplicate node name {name!r}")
        self.nodes[name] = spec
        return name


class SymArray:
    """A node of the recorded graph: name, shape, dtype.  Mirrors ``LazyArray``
    (/root/reference/pkg/src/laze/frontend.py:158-250)."""

    __array_priority__ = 100.0

    def __init__(self, ctx, scope, name, shape, dtype):
        self.ctx, self.scope, self.name, self.shape, self.dtype = ctx, scope, name, tuple(int(s) for s in shape), dtype

    @property
    def ndim(self):
        return len(self.shape)

    def reshape(self, *shape):
        return self.ctx.np.reshape(self, shape[0] if len(shape) == 1 and not isinstance(shape[0], int) else shape)

    def tagged(self, axis, key, value=None):
        return self

    def __getitem__(self, sel):
        return self.ctx._index(self, sel)

    def __neg__(self):
        return self.ctx._unary("neg", self)

    def __abs__(self):
        return self.ctx._unary("abs", self)


def _install_operators():
    table = {"add": "add", "sub": "sub", "mul": "mul", "truediv": "truediv", "floordiv": "floordiv", "mod": "mod",
             "pow": "pow", "lt": "lt", "le": "le", "gt": "gt", "ge": "ge"}
    for dunder, op in table.items():
        setattr(SymArray, f"__{dunder}__", lambda self, other, op=op: self.ctx._binary(op, self, other))
        if dunder in ("add", "sub", "mul", "truediv", "floordiv", "mod", "pow"):
            setattr(SymArray, f"__r{dunder}__", lambda self, other, op=op: self.ctx._binary(op, other, self))


_install_operators()


class _Ops:
    """The op namespace of /root/reference/pkg/src/laze/frontend.py:257-302."""

    def __init__(self, ctx):
        c = self._c = ctx
        for name, op in [("add", "add"), ("subtract", "sub"), ("multiply", "mul"), ("divide", "truediv"), ("power", "pow"),
                         ("maximum", "max"), ("minimum", "min"), ("greater", "gt"), ("greater_equal", "ge"),
                         ("less", "lt"), ("less_equal", "le"), ("equal", "eq"), ("not_equal", "ne")]:
            setattr(self, name, lambda a, b, op=op: c._binary(op, a, b))
        for name, op in [("negative", "neg"), ("abs", "abs"), ("sqrt", "sqrt"), ("exp", "exp"), ("log", "log")]:
            setattr(self, name, lambda a, op=op: c._unary(op, a))

    def where(self, cond, a, b):
        return self._c._where(cond, a, b)

    def reshape(self, a, shape):
        c = self._c
        a = c._as_array(a)
        shape = [int(s) for s in (shape if isinstance(shape, (tuple, list)) else (shape,))]
        size = int(np.prod(a.shape, dtype=np.int64))
        if -1 in shape:                                          # frontend.py:689-707
            known = int(np.prod([s for s in shape if s != -1], dtype=np.int64))
            shape[shape.index(-1)] = size // known if known else 0
        if int(np.prod(shape, dtype=np.int64)) != size:
            raise errors.ShapeMismatch(f"cannot reshape {a.shape} to {tuple(shape)}")
        return c._node({"kind": "reshape", "array": a.name, "shape": list(shape)}, shape, a.dtype, a.scope)

    def concatenate(self, arrays, axis=0):
        c = self._c
        arrays = [c._as_array(a) for a in arrays]
        shape = list(arrays[0].shape)
        shape[axis] = sum(a.shape[axis] for a in arrays)
        return c._node({"kind": "concatenate", "axis": int(axis), "arrays": [a.name for a in arrays]}, shape,
                       arrays[0].dtype, arrays[0].scope)

    def stack(self, arrays, axis=0):
        c = self._c
        arrays = [c._as_array(a) for a in arrays]
        shape = list(arrays[0].shape)
        shape.insert(axis, len(arrays))
        return c._node({"kind": "stack", "axis": int(axis), "arrays": [a.name for a in arrays]}, shape,
                       arrays[0].dtype, arrays[0].scope)

    def einsum(self, subscripts, *args):
        c = self._c
        args = [c._as_array(a) for a in args]
        lhs, out = subscripts.replace(" ", "").split("->")
        extent = {}
        for term, a in zip(lhs.split(","), args):
            if len(term) != a.ndim:
                raise errors.ShapeMismatch(f"einsum term {term!r} does not match an operand of rank {a.ndim}")
            for letter, n in zip(term, a.shape):
                if extent.setdefault(letter, n) != n:
                    raise errors.ShapeMismatch(f"einsum index {letter!r} has extents {extent[letter]} and {n}")
        return c._node({"kind": "einsum", "subscripts": subscripts, "args": [a.name for a in args]},
                       [extent[letter] for letter in out], c._result_dtype("mul", args), args[0].scope)

    def sum(self, a, axis=None):
        a = self._c._as_array(a)
        letters = "abcdefgh"[:a.ndim]
        axes = range(a.ndim) if axis is None else [axis % a.ndim]
        return self.einsum(f"{letters}->{''.join(l for k, l in enumerate(letters) if k not in axes)}", a)


class GraphExportContext:
    """Records the operator program; ``to_doc`` returns the reference CLI's program document."""

    mode = "lazy"

    def __init__(self, name="program"):
        self.name = name
        self.top = _Scope()
        self._scope = self.top
        self.functions: dict[str, dict] = {}
        self._fkeys: dict = {}
        self.bindings: dict[str, list] = {}
        self.np = _Ops(self)

    # {{{ creation (frontend.py:327-343)

    def placeholder(self, name, shape, dtype="f64", value=None):
        a = SymArray(self, self._scope, self._scope.add({"kind": "placeholder", "shape": [int(s) for s in shape], "dtype": dtype},
                                                        name), shape, dtype)
        if value is not None:
            self.bindings[name] = np.asarray(value).tolist()
        return a

    def from_numpy(self, value):
        value = np.asarray(value)
        if value.dtype not in _DT:
            raise errors.DTypeMismatch(f"unsupported element type: {value.dtype}")
        dt = _DT[value.dtype]
        return self._node({"kind": "data", "value": value.tolist(), "dtype": dt}, value.shape, dt, self._scope, prefix="_d")

    def to_numpy(self, value):
        raise errors.LazeError("GraphExportContext records a program; it has no values")

    def freeze(self, what):
        return what

    def compile(self, f):
        return f

    # }}}

    # {{{ recording

    def _node(self, spec, shape, dtype, scope, prefix=None):
        if scope is not self._scope:
            raise errors.LazeError("an outlined function body used an array of the enclosing program (pass it as an argument)")
        return SymArray(self, scope, scope.add(spec), shape, dtype)

    def _as_array(self, x):
        if isinstance(x, SymArray):
            return x
        if hasattr(x, "data") and isinstance(getattr(x, "data"), SymArray):       # DOFArray
            return x.data
        if isinstance(x, (list, tuple)) and x and all(isinstance(v, SymArray) for v in x):
            return self.np.stack(list(x))
        return self.from_numpy(np.asarray(x))

    @staticmethod
    def _is_scalar(x):
        return isinstance(x, (bool, int, float, np.bool_, np.integer, np.floating))

    def _result_dtype(self, op, arrays):
        if op in _COMPARE:
            return "bool"
        kinds = {a.dtype for a in arrays}
        if "f64" in kinds or op == "truediv":
            return "f64"
        if "f32" in kinds:
            return "f32"
        return "i64" if "i64" in kinds else "bool"

    def _pointwise(self, op, operands, render):
        """One ``expression`` node; python scalars are weak literals (/root/reference/pkg/src/laze/adfg.py:876-932)."""
        arrays = [o for o in operands if isinstance(o, SymArray)]
        shape = np.broadcast_shapes(*[a.shape for a in arrays]) if arrays else ()
        rank = len(shape)
        inputs, texts = [], []
        for o in operands:
            if isinstance(o, SymArray):
                if o.name not in inputs:
                    inputs.append(o.name)
                if o.ndim == 0:
                    texts.append(f"{o.name}[()]")
                else:
                    idx = ["0" if (n == 1 and shape[rank - o.ndim + k] != 1) else f"i{rank - o.ndim + k}"
                           for k, n in enumerate(o.shape)]
                    texts.append(f"{o.name}[{', '.join(idx)}]")
            else:
                v = o.item() if isinstance(o, np.generic) else o
                texts.append(repr(v) if not (isinstance(v, (int, float)) and not isinstance(v, bool) and v < 0) else f"({v!r})")
        spec = {"kind": "expression", "shape": [int(s) for s in shape], "inputs": inputs, "expr": render(*texts)}
        return self._node(spec, shape, self._result_dtype(op, arrays), arrays[0].scope)

    def _coerce(self, x):
        return x if (isinstance(x, SymArray) or self._is_scalar(x)) else self._as_array(x)

    def _binary(self, op, a, b):
        a, b = self._coerce(a), self._coerce(b)
        if op in ("min", "max"):
            return self._pointwise(op, [a, b], lambda x, y: f"{op}({x}, {y})")
        return self._pointwise(op, [a, b], lambda x, y: f"({x}) {_BIN_SYMBOL[op]} ({y})")

    def _unary(self, op, a):
        a = self._coerce(a)
        return self._pointwise(op, [a], (lambda x: f"-({x})") if op == "neg" else (lambda x: f"{op}({x})"))

    def _where(self, cond, a, b):
        cond, a, b = self._coerce(cond), self._coerce(a), self._coerce(b)
        out = self._pointwise("where", [cond, a, b], lambda c, x, y: f"where({c}, {x}, {y})")
        out.dtype = self._result_dtype("add", [v for v in (a, b) if isinstance(v, SymArray)] or [out])
        return out

    def _index(self, a, sel):
        """``Indexing``: ints, slices with positive step and at most one i64 index array
        (/root/reference/pkg/src/laze/adfg.py:502-560)."""
        sel = sel if isinstance(sel, tuple) else (sel,)
        if len(sel) > a.ndim:
            raise errors.BadSubscript(f"too many subscripts for an array of rank {a.ndim}")
        selectors, shape = [], []
        for axis, s in enumerate(sel):
            n = a.shape[axis]
            if isinstance(s, (int, np.integer)):
                s = int(s) + (n if s < 0 else 0)
                if not 0 <= s < n:
                    raise errors.BadSubscript(f"index {s} outside [0, {n})")
                selectors.append(s)
            elif isinstance(s, slice):
                start, stop, step = s.indices(n)
                if step <= 0:
                    raise errors.BadSubscript("slices need a positive step")
                selectors.append({"slice": [start, stop, step]})
                shape.append(max(0, (stop - start + step - 1) // step))
            elif isinstance(s, SymArray):
                if s.dtype != "i64":
                    raise errors.DTypeMismatch("index arrays must be i64")
                selectors.append({"array": s.name})
                shape.extend(s.shape)
            else:
                raise errors.BadSubscript(f"unsupported subscript {s!r}")
        for n in a.shape[len(sel):]:                          # the node carries one selector per axis (adfg.py:516-520)
            selectors.append({"slice": [0, int(n), 1]})
            shape.append(n)
        return self._node({"kind": "index", "array": a.name, "selectors": selectors}, shape, a.dtype, a.scope)

    # }}}

    # {{{ outlined functions (frontend.py:488-519)

    def outline(self, f):
        def call(*args):
            args = [self._as_array(a) for a in args]
            key = (f.__name__, getattr(f, "dg_dim", None), tuple((a.shape, a.dtype) for a in args))
            if key not in self._fkeys:
                if self._scope is not self.top:
                    raise errors.LazeError("cannot serialize calls nested inside function bodies")
                body = _Scope()
                self._scope = body
                try:
                    params = {f"_p{k}": {"shape": list(a.shape), "dtype": a.dtype} for k, a in enumerate(args)}
                    formal = [SymArray(self, body, f"_p{k}", a.shape, a.dtype) for k, a in enumerate(args)]
                    res = f(*formal)
                finally:
                    self._scope = self.top
                res = res if isinstance(res, dict) else {"out": res}
                label = f"_f{len(self.functions)}"
                self.functions[label] = {"name": f.__name__, "parameters": params, "nodes": body.nodes,
                                         "returns": {k: v.name for k, v in res.items()}}
                self._fkeys[key] = (label, {k: (v.shape, v.dtype) for k, v in res.items()})
            label, results = self._fkeys[key]
            names = sorted(results)
            spec = {"kind": "call", "function": label, "args": {f"_p{k}": a.name for k, a in enumerate(args)}}
            first = self._node(spec, *results[names[0]], self.top)          # the call node stands for its first result
            out = {names[0]: first}
            for rname in names[1:]:
                out[rname] = self._node({"kind": "result", "call": first.name, "result": rname}, *results[rname], self.top)
            return out if (len(out) > 1 or "out" not in out) else out["out"]
        call.__name__ = f.__name__
        return call

    # }}}

    def to_doc(self, outputs) -> dict:
        """The program document (cli.py:322-335): ``{"name", "nodes", "outputs", "functions", "bindings"}``."""
        if not isinstance(outputs, dict):
            outputs = {"out": outputs}
        doc = {"name": self.name, "nodes": self.top.nodes,
               "outputs": {k: self._as_array(v).name for k, v in outputs.items()}}
        if self.functions:
            doc["functions"] = self.functions
        if self.bindings:
            doc["bindings"] = self.bindings
        return doc


def export_rhs_program(mesh, order, q0, equations="ns", name=None, **phys) -> dict:
    """The right-hand side of ``equations`` ("ns" = flux arrangement, "ns_grad_form", "euler", "multispecies") on
    ``mesh`` as a program document with the state as the placeholder ``q`` bound to ``q0``."""
    from .discretization import DGDiscretization
    from .dofarray import DOFArray
    from .operators import EulerOperator, NavierStokesOperator
    ctx = GraphExportContext(name or f"dg_{equations}_rhs")
    d = DGDiscretization(ctx, mesh, order)
    q = DOFArray(ctx, ctx.placeholder("q", np.shape(q0), "f64", value=q0))
    if equations == "multispecies":
        from .multispecies import MultispeciesOperator
        out = MultispeciesOperator(d, **phys).rhs(q)
    elif equations == "euler":
        out = EulerOperator(d, **phys).rhs(q)
    else:
        op = NavierStokesOperator(d, **phys)
        out = op.rhs(q) if equations == "ns" else op.rhs_grad_form(q)
    return ctx.to_doc({"rhs": out.data})
