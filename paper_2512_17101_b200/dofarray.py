"""Minimal ``DOFArray``: element-major nodal data bound to an array context.

NEW SURFACE -- the reference package has no ``DOFArray`` (the identifier does not occur
under /root/reference/pkg).  The layout follows the paper's description only:
per-element nodal values, one row per element, with the
axis meaning "element / DOF inside an element" attached by the DG layer
(tag keys in /root/reference/SPEC.md:34).

``data`` has shape ``(..., nelements, ndofs)``; leading axes are components (conserved
fields, gradient directions).  Arithmetic is delegated to the wrapped arrays, so it runs
on whatever the array context hands out (NumPy arrays, ``laze.LazyArray``, or B200
``DeviceArray``).
"""
from __future__ import annotations

import numbers


class DOFArray:
    __slots__ = ("actx", "data")
    __array_priority__ = 1000   # make ndarray.__op__ defer to us

    def __init__(self, actx, data):
        self.actx = actx
        self.data = data

    # {{{ structure

    @property
    def shape(self):
        return tuple(self.data.shape)

    @property
    def nelements(self) -> int:
        return self.shape[-2]

    @property
    def ndofs(self) -> int:
        return self.shape[-1]

    def __len__(self):
        return self.shape[0]

    def __getitem__(self, comp):
        """Component selection on the leading axes only (keeps element/dof axes)."""
        if not isinstance(comp, tuple):
            comp = (comp,)
        if len(comp) > len(self.shape) - 2:
            raise IndexError("DOFArray subscripts address component axes only")
        out = self.data
        for c in comp:
            if not isinstance(c, numbers.Integral):
                raise IndexError("component subscripts must be integers")
            out = out[int(c)]
        return DOFArray(self.actx, out)

    def tagged(self):
        """Attach the reference's axis-tag vocabulary when the array supports it
        (/root/reference/pkg/src/laze/frontend.py:182-187)."""
        d = self.data
        if hasattr(d, "tagged"):
            rank = len(d.shape)
            d = d.tagged(rank - 2, "kind", "element").tagged(rank - 1, "kind", "dof")
        return DOFArray(self.actx, d)

    # }}}

    # {{{ arithmetic

    @staticmethod
    def _raw(x):
        return x.data if isinstance(x, DOFArray) else x

    def _new(self, data):
        return DOFArray(self.actx, data)

    def __add__(self, o): return self._new(self.data + self._raw(o))
    def __radd__(self, o): return self._new(self._raw(o) + self.data)
    def __sub__(self, o): return self._new(self.data - self._raw(o))
    def __rsub__(self, o): return self._new(self._raw(o) - self.data)
    def __mul__(self, o): return self._new(self.data * self._raw(o))
    def __rmul__(self, o): return self._new(self._raw(o) * self.data)
    def __truediv__(self, o): return self._new(self.data / self._raw(o))
    def __rtruediv__(self, o): return self._new(self._raw(o) / self.data)
    def __neg__(self): return self._new(-self.data)

    # }}}

    def to_numpy(self):
        return self.actx.to_numpy(self.data)

    def __repr__(self):
        return f"DOFArray(shape={self.shape})"
