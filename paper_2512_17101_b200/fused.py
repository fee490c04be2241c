"""Fused implementations of the outlined DG functions, keyed by function name.

``B200ArrayContext.outline(f)`` looks ``f.__name__`` up here.  Each implementation receives the
same positional arrays the reference would bind to the ``FunctionDefinition`` parameters
``_p0, _p1, ...`` (/root/reference/pkg/src/laze/frontend.py:501) and returns the array(s) the
body would return, but computes them with one (or, for nothing here, more) fused sm_100a kernel
through the C ABI (include/dgb200.h).  The per-mesh discretisation handle is created on first
use from the argument arrays themselves and cached on their identity; creating it validates
the int64 face maps on the device (range check + conformity) exactly once.
"""
from __future__ import annotations

import ast
import ctypes as C
import hashlib
import inspect
import json
import os
import textwrap
import types
import warnings

import numpy as np

from . import _cabi, errors
from .dg.simplex import simplex_element

_ORDER_OF_NP = {(2, 3): 1, (2, 6): 2, (2, 10): 3, (2, 15): 4, (3, 4): 1, (3, 10): 2, (3, 20): 3, (3, 35): 4}


class _Disc:
    def __init__(self, lib, handle, keep):
        self.lib, self.handle, self.keep = lib, handle, keep

    def __del__(self):
        try:
            if self.handle:
                self.lib.dgb_disc_destroy(self.handle)
        except Exception:
            pass


def _f64(actx, a, what):
    from .actx import F64
    if a.dtype_code != F64:
        raise errors.DTypeMismatch(f"{what} must be f64")
    return actx._contiguous(a)


def _i64(actx, a, what):
    from .actx import I64
    if a.dtype_code != I64:
        raise errors.DTypeMismatch(f"{what} must be i64")
    return actx._contiguous(a)


def get_disc(actx, dim, q, nghost, Sw, drdx, lift, normals, fscale, vmap_m, vmap_p, bc_kind, nspecies=0) -> _Disc:
    key = (dim, nghost, id(Sw), id(drdx), id(lift), id(normals), id(fscale), id(vmap_m), id(vmap_p), id(bc_kind))
    disc = actx._discs.get(key)
    if disc is not None:
        return disc
    C_, E, Np = q.shape
    if C_ != dim + 2 + nspecies:
        raise errors.ShapeMismatch(f"state has {C_} fields, expected {dim + 2 + nspecies}")
    order = _ORDER_OF_NP.get((dim, Np))
    if order is None:
        raise errors.ShapeMismatch(f"no simplex element with dim={dim}, Np={Np} (orders 1..4 are built)")
    el = simplex_element(dim, order)
    Nf, Nfp = el.Nf, el.Nfp
    expect = {"Sw": (Sw, (dim, Np, Np)), "drdx": (drdx, (dim, dim, E)), "lift": (lift, (Np, Nf * Nfp)),
              "normals": (normals, (dim, E, Nf, 1)), "fscale": (fscale, (E, Nf, 1)),
              "vmap_m": (vmap_m, (E * Nf * Nfp,)), "vmap_p": (vmap_p, (E * Nf * Nfp,)),
              "bc_kind": (bc_kind, (E, Nf, 1))}
    for name, (arr, shape) in expect.items():
        if tuple(arr.shape) != shape:
            raise errors.BindingMismatch(f"{name} has shape {tuple(arr.shape)}, expected {shape}")
    Sw_h = np.ascontiguousarray(Sw.host_value(), dtype=np.float64)
    lift_h = np.ascontiguousarray(lift.host_value(), dtype=np.float64)
    fn_h = np.ascontiguousarray(el.face_nodes, dtype=np.int64)
    fp_h = np.ascontiguousarray(el.face_perms, dtype=np.int64)
    keep = [_f64(actx, drdx, "drdx"), _f64(actx, normals, "normals"), _f64(actx, fscale, "fscale"),
            _i64(actx, vmap_m, "vmap_m"), _i64(actx, vmap_p, "vmap_p"), _i64(actx, bc_kind, "bc_kind"),
            Sw, drdx, lift, normals, fscale, vmap_m, vmap_p, bc_kind]
    handle = C.c_void_p()
    _cabi.check(actx.lib.dgb_disc_create(
        C.byref(handle), dim, order, E, nghost,
        Sw_h.ctypes.data, lift_h.ctypes.data, fn_h.ctypes.data, fp_h.ctypes.data,
        keep[0].ptr, keep[1].ptr, keep[2].ptr, keep[3].ptr, keep[4].ptr, keep[5].ptr, actx._st), "face index maps")
    actx.launch_count += 1
    disc = _Disc(actx.lib, handle, keep)
    disc.dim, disc.order, disc.E, disc.Np, disc.Nf, disc.Nfp, disc.G = dim, order, E, Np, Nf, Nfp, nghost
    actx._discs[key] = disc
    # dg_ns_div does not take drdx (the metric is already inside the flux planes): second index without it
    actx._discs[("nodrdx",) + key[:3] + key[4:]] = disc
    return disc


def _host_vec(arr, n):
    v = np.ascontiguousarray(np.asarray(arr.host_value(), dtype=np.float64).reshape(-1))
    if v.size != n:
        raise errors.BindingMismatch(f"expected {n} parameters, got {v.size}")
    return v


def _ghost_ptr(actx, ghost, lead, Np):
    if ghost is None:
        return 0, None, None
    g = _f64(actx, ghost, "ghost")
    if g.shape[:-2] != lead or g.shape[-1] != Np:
        raise errors.BindingMismatch(f"ghost array has shape {g.shape}")
    return g.shape[-2], g, g.ptr


def _euler(actx, f, q, ghost, Sw, drdx, lift, normals, fscale, vmap_m, vmap_p, bc_kind, qfar, phys, epi=None):
    dim = f.dg_dim
    q = _f64(actx, q, "q")
    G, g, gptr = _ghost_ptr(actx, ghost, (dim + 2,), q.shape[-1])
    disc = get_disc(actx, dim, q, G, Sw, drdx, lift, normals, fscale, vmap_m, vmap_p, bc_kind)
    qf, ph = _host_vec(qfar, dim + 2), _host_vec(phys, 4)
    out = actx.empty(q.shape)
    _cabi.check(actx.lib.dgb_euler_rhs(disc.handle, q.ptr, gptr, out.ptr, qf.ctypes.data, ph.ctypes.data,
                                       actx._st), "dg_euler_rhs")
    actx.launch_count += 1
    return out


def dg_euler_rhs(actx, f, *args):
    if len(args) == 11:
        q, Sw, drdx, lift, normals, fscale, vmap_m, vmap_p, bc_kind, qfar, phys = args
        ghost = None
    elif len(args) == 12:
        q, ghost, Sw, drdx, lift, normals, fscale, vmap_m, vmap_p, bc_kind, qfar, phys = args
    else:
        raise errors.BindingMismatch(f"dg_euler_rhs takes 11 or 12 arrays, got {len(args)}")
    return _euler(actx, f, q, ghost, Sw, drdx, lift, normals, fscale, vmap_m, vmap_p, bc_kind, qfar, phys)


def dg_ns_grad(actx, f, *args):
    if len(args) == 10:
        q, Sw, drdx, lift, normals, fscale, vmap_m, vmap_p, bc_kind, qfar = args
        ghost = None
    elif len(args) == 11:
        q, ghost, Sw, drdx, lift, normals, fscale, vmap_m, vmap_p, bc_kind, qfar = args
    else:
        raise errors.BindingMismatch(f"dg_ns_grad takes 10 or 11 arrays, got {len(args)}")
    dim = f.dg_dim
    q = _f64(actx, q, "q")
    G, g, gptr = _ghost_ptr(actx, ghost, (dim + 2,), q.shape[-1])
    disc = get_disc(actx, dim, q, G, Sw, drdx, lift, normals, fscale, vmap_m, vmap_p, bc_kind)
    qf = _host_vec(qfar, dim + 2)
    out = actx.empty((dim,) + q.shape)
    _cabi.check(actx.lib.dgb_ns_grad(disc.handle, q.ptr, gptr, out.ptr, qf.ctypes.data, actx._st), "dg_ns_grad")
    actx.launch_count += 1
    return out


def dg_ns_rhs(actx, f, *args):
    if len(args) == 12:
        q, gq, Sw, drdx, lift, normals, fscale, vmap_m, vmap_p, bc_kind, qfar, phys = args
        ghost = gghost = None
    elif len(args) == 14:
        q, gq, ghost, gghost, Sw, drdx, lift, normals, fscale, vmap_m, vmap_p, bc_kind, qfar, phys = args
    else:
        raise errors.BindingMismatch(f"dg_ns_rhs takes 12 or 14 arrays, got {len(args)}")
    dim = f.dg_dim
    q = _f64(actx, q, "q")
    gq = _f64(actx, gq, "grad q")
    if gq.shape != (dim,) + q.shape:
        raise errors.BindingMismatch(f"grad q has shape {gq.shape}, expected {(dim,) + q.shape}")
    G, g, gptr = _ghost_ptr(actx, ghost, (dim + 2,), q.shape[-1])
    GG, gg, ggptr = _ghost_ptr(actx, gghost, (dim, dim + 2), q.shape[-1])
    if GG != G:
        raise errors.BindingMismatch("ghost arrays of q and grad q disagree in size")
    disc = get_disc(actx, dim, q, G, Sw, drdx, lift, normals, fscale, vmap_m, vmap_p, bc_kind)
    qf, ph = _host_vec(qfar, dim + 2), _host_vec(phys, 4)
    out = actx.empty(q.shape)
    _cabi.check(actx.lib.dgb_ns_rhs(disc.handle, q.ptr, gq.ptr, gptr, ggptr, out.ptr, qf.ctypes.data,
                                    ph.ctypes.data, actx._st), "dg_ns_rhs")
    actx.launch_count += 1
    return out


def _rk_common(actx, q, x1, x2, coef):
    x1 = _f64(actx, x1, "x1")
    x2 = _f64(actx, x2, "x2")
    if x1.shape != q.shape or x2.shape != q.shape:
        raise errors.BindingMismatch("RK operands must have the shape of the state")
    rk = _host_vec(coef, 4)
    return x1, x2, rk, actx.empty(q.shape), actx.empty(q.shape)


def dg_euler_rhs_rk(actx, f, q, x1, x2, coef, Sw, drdx, lift, normals, fscale, vmap_m, vmap_p, bc_kind, qfar, phys):
    dim = f.dg_dim
    q = _f64(actx, q, "q")
    disc = get_disc(actx, dim, q, 0, Sw, drdx, lift, normals, fscale, vmap_m, vmap_p, bc_kind)
    qf, ph = _host_vec(qfar, dim + 2), _host_vec(phys, 4)
    x1, x2, rk, o1, o2 = _rk_common(actx, q, x1, x2, coef)
    _cabi.check(actx.lib.dgb_euler_rhs_rk(disc.handle, q.ptr, None, x1.ptr, o1.ptr, x2.ptr, o2.ptr, rk.ctypes.data,
                                          qf.ctypes.data, ph.ctypes.data, actx._st), "dg_euler_rhs_rk")
    actx.launch_count += 1
    return {"out1": o1, "out2": o2}


def dg_ns_rhs_rk(actx, f, q, gq, x1, x2, coef, Sw, drdx, lift, normals, fscale, vmap_m, vmap_p, bc_kind, qfar, phys):
    dim = f.dg_dim
    q = _f64(actx, q, "q")
    gq = _f64(actx, gq, "grad q")
    disc = get_disc(actx, dim, q, 0, Sw, drdx, lift, normals, fscale, vmap_m, vmap_p, bc_kind)
    qf, ph = _host_vec(qfar, dim + 2), _host_vec(phys, 4)
    x1, x2, rk, o1, o2 = _rk_common(actx, q, x1, x2, coef)
    _cabi.check(actx.lib.dgb_ns_rhs_rk(disc.handle, q.ptr, gq.ptr, None, None, x1.ptr, o1.ptr, x2.ptr, o2.ptr,
                                       rk.ctypes.data, qf.ctypes.data, ph.ctypes.data, actx._st), "dg_ns_rhs_rk")
    actx.launch_count += 1
    return {"out1": o1, "out2": o2}


def flux_planes(dim: int) -> int:
    """Planes of the array ``dg_ns_flux`` returns: dim + 1 groups of C = dim + 2 flux planes and the wave speed."""
    return (dim + 1) * (dim + 2) + 1


def _bind_jacobian(actx, disc, jac, facemat=None):
    """Bind the volume Jacobian argument to the handle (once) -- dgb_disc_set_jacobian."""
    if getattr(disc, "jac_id", None) == id(jac):
        return
    j = _f64(actx, jac, "jac")
    if tuple(j.shape) != (disc.E,):
        raise errors.BindingMismatch(f"jac has shape {tuple(j.shape)}, expected {(disc.E,)}")
    _cabi.check(actx.lib.dgb_disc_set_jacobian(disc.handle, j.ptr, actx._st), "dgb_disc_set_jacobian")
    actx.launch_count += 1
    disc.keep += [j, jac]
    disc.jac_id = id(jac)


def _check_facemat(disc, facemat, facemat_p):
    """The kernels use the simplex identity behind ``facemat`` (face 0 = sum of the reference
    gradients, face f = minus gradient f-1) structurally; refuse anything else."""
    if getattr(disc, "facemat_ok", None) == (id(facemat), id(facemat_p)):
        return
    dim, Nf = disc.dim, disc.Nf
    want = np.zeros((dim + 1, Nf))
    want[dim, 0] = 1.0
    for r in range(dim):
        want[r, r + 1] = -1.0
    got = np.asarray(facemat.host_value(), dtype=np.float64).reshape(dim + 1, Nf)
    if not np.array_equal(got, want):
        raise errors.BindingMismatch("facemat is not the simplex face/plane-group selection matrix")
    if tuple(facemat_p.shape) != (dim + 1, disc.E, Nf, 1):
        raise errors.BindingMismatch(f"facemat_p has shape {tuple(facemat_p.shape)}")
    disc.facemat_ok = (id(facemat), id(facemat_p))


def dg_ns_flux(actx, f, *args):
    if len(args) == 12:
        q, Sw, drdx, jac, lift, normals, fscale, vmap_m, vmap_p, bc_kind, qfar, phys = args
        ghost = None
    elif len(args) == 13:
        q, ghost, Sw, drdx, jac, lift, normals, fscale, vmap_m, vmap_p, bc_kind, qfar, phys = args
    else:
        raise errors.BindingMismatch(f"dg_ns_flux takes 12 or 13 arrays, got {len(args)}")
    dim = f.dg_dim
    q = _f64(actx, q, "q")
    G, g, gptr = _ghost_ptr(actx, ghost, (dim + 2,), q.shape[-1])
    disc = get_disc(actx, dim, q, G, Sw, drdx, lift, normals, fscale, vmap_m, vmap_p, bc_kind)
    _bind_jacobian(actx, disc, jac)
    qf, ph = _host_vec(qfar, dim + 2), _host_vec(phys, 4)
    out = actx.empty((flux_planes(dim),) + tuple(q.shape[1:]))
    _cabi.check(actx.lib.dgb_ns_flux(disc.handle, q.ptr, gptr, out.ptr, qf.ctypes.data, ph.ctypes.data, actx._st),
                "dg_ns_flux")
    actx.launch_count += 1
    return out


def _div_common(actx, f, q, T, ghost, Tghost, Sw, jac, lift, normals, fscale, facemat, facemat_p, vmap_m, vmap_p,
                bc_kind):
    dim = f.dg_dim
    q = _f64(actx, q, "q")
    T = _f64(actx, T, "T")
    npl = flux_planes(dim)
    if tuple(T.shape) != (npl,) + tuple(q.shape[1:]):
        raise errors.BindingMismatch(f"flux planes have shape {tuple(T.shape)}, expected {(npl,) + tuple(q.shape[1:])}")
    G, g, gptr = _ghost_ptr(actx, ghost, (dim + 2,), q.shape[-1])
    TG, tg, tgptr = _ghost_ptr(actx, Tghost, (npl,), q.shape[-1])
    if TG != G:
        raise errors.BindingMismatch("ghost arrays of q and of the flux planes disagree in size")
    # dg_ns_div does not receive drdx; the handle was created by dg_ns_flux of the same discretisation
    disc = actx._discs.get(("nodrdx", dim, G, id(Sw), id(lift), id(normals), id(fscale), id(vmap_m), id(vmap_p),
                            id(bc_kind)))
    if disc is None:
        raise errors.BindingMismatch("dg_ns_div: no discretisation handle for these arrays (call dg_ns_flux first)")
    _bind_jacobian(actx, disc, jac)
    _check_facemat(disc, facemat, facemat_p)
    return q, T, gptr, tgptr, disc, (g, tg)


def dg_ns_div(actx, f, *args):
    if len(args) == 14:
        q, T, Sw, jac, lift, normals, fscale, facemat, facemat_p, vmap_m, vmap_p, bc_kind, qfar, phys = args
        ghost = Tghost = None
    elif len(args) == 16:
        q, T, ghost, Tghost, Sw, jac, lift, normals, fscale, facemat, facemat_p, vmap_m, vmap_p, bc_kind, qfar, phys = args
    else:
        raise errors.BindingMismatch(f"dg_ns_div takes 14 or 16 arrays, got {len(args)}")
    q, T, gptr, tgptr, disc, keep = _div_common(actx, f, q, T, ghost, Tghost, Sw, jac, lift, normals, fscale, facemat,
                                                facemat_p, vmap_m, vmap_p, bc_kind)
    qf, ph = _host_vec(qfar, f.dg_dim + 2), _host_vec(phys, 4)
    out = actx.empty(q.shape)
    _cabi.check(actx.lib.dgb_ns_div(disc.handle, q.ptr, T.ptr, gptr, tgptr, out.ptr, qf.ctypes.data, ph.ctypes.data,
                                    actx._st), "dg_ns_div")
    actx.launch_count += 1
    return out


def dg_ns_div_rk(actx, f, q, T, x1, x2, coef, Sw, jac, lift, normals, fscale, facemat, facemat_p, vmap_m, vmap_p,
                 bc_kind, qfar, phys):
    q, T, gptr, tgptr, disc, keep = _div_common(actx, f, q, T, None, None, Sw, jac, lift, normals, fscale, facemat,
                                                facemat_p, vmap_m, vmap_p, bc_kind)
    qf, ph = _host_vec(qfar, f.dg_dim + 2), _host_vec(phys, 4)
    x1, x2, rk, o1, o2 = _rk_common(actx, q, x1, x2, coef)
    _cabi.check(actx.lib.dgb_ns_div_rk(disc.handle, q.ptr, T.ptr, None, None, x1.ptr, o1.ptr, x2.ptr, o2.ptr,
                                       rk.ctypes.data, qf.ctypes.data, ph.ctypes.data, actx._st), "dg_ns_div_rk")
    actx.launch_count += 1
    return {"out1": o1, "out2": o2}


# {{{ element sub-ranges (halo.py overlaps the interior range with the exchange)

def _op_disc(actx, op, q, nghost):
    d = op.dcoll
    disc = get_disc(actx, op.dim, q, nghost, d.Sw, d.drdx, d.lift, d.normals, d.fscale, d.vmap_m, d.vmap_p, d.bc_kind)
    return disc


def euler_rhs_range(actx, op, q, ghost, out, lo, hi):
    """``out[:, lo:hi] = dg_euler_rhs(q)[:, lo:hi]`` (dgb_euler_rhs_range)."""
    q = _f64(actx, q, "q")
    G, g, gptr = _ghost_ptr(actx, ghost, (op.dim + 2,), q.shape[-1])
    disc = _op_disc(actx, op, q, G)
    _cabi.check(actx.lib.dgb_euler_rhs_range(disc.handle, q.ptr, gptr, out.ptr, op.qfar_host.ctypes.data,
                                             op.phys_host.ctypes.data, int(lo), int(hi), actx._st), "dg_euler_rhs (range)")
    actx.launch_count += 1


def ns_flux_range(actx, op, q, ghost, T, lo, hi):
    """``T[:, lo:hi] = dg_ns_flux(q)[:, lo:hi]`` (dgb_ns_flux_range)."""
    q = _f64(actx, q, "q")
    G, g, gptr = _ghost_ptr(actx, ghost, (op.dim + 2,), q.shape[-1])
    disc = _op_disc(actx, op, q, G)
    _bind_jacobian(actx, disc, op.dcoll.jac)
    _cabi.check(actx.lib.dgb_ns_flux_range(disc.handle, q.ptr, gptr, T.ptr, op.qfar_host.ctypes.data,
                                           op.phys_host.ctypes.data, int(lo), int(hi), actx._st), "dg_ns_flux (range)")
    actx.launch_count += 1


def ns_div_range(actx, op, q, T, ghost, Tghost, out, lo, hi):
    """``out[:, lo:hi] = dg_ns_div(q, T)[:, lo:hi]`` (dgb_ns_div_range)."""
    q = _f64(actx, q, "q")
    npl = flux_planes(op.dim)
    G, g, gptr = _ghost_ptr(actx, ghost, (op.dim + 2,), q.shape[-1])
    TG, tg, tgptr = _ghost_ptr(actx, Tghost, (npl,), q.shape[-1])
    disc = _op_disc(actx, op, q, G)
    _bind_jacobian(actx, disc, op.dcoll.jac)
    _check_facemat(disc, op.dcoll.facemat, op.dcoll.facemat_p)
    _cabi.check(actx.lib.dgb_ns_div_range(disc.handle, q.ptr, T.ptr, gptr, tgptr, out.ptr, op.qfar_host.ctypes.data,
                                          op.phys_host.ctypes.data, int(lo), int(hi), actx._st), "dg_ns_div (range)")
    actx.launch_count += 1

def ns_div_rk_range(actx, op, q, T, ghost, Tghost, x1, out1, x2, out2, coef, lo, hi):
    """``out1[:, lo:hi] = a1 x1 + b1 rhs``, ``out2[:, lo:hi] = a2 x2 + b2 rhs`` with ``rhs = dg_ns_div(q, T)``
    (dgb_ns_div_rk_range): the RK stage update fused into pass 2 of a partitioned right-hand side."""
    q = _f64(actx, q, "q")
    npl = flux_planes(op.dim)
    G, g, gptr = _ghost_ptr(actx, ghost, (op.dim + 2,), q.shape[-1])
    TG, tg, tgptr = _ghost_ptr(actx, Tghost, (npl,), q.shape[-1])
    disc = _op_disc(actx, op, q, G)
    _bind_jacobian(actx, disc, op.dcoll.jac)
    _check_facemat(disc, op.dcoll.facemat, op.dcoll.facemat_p)
    x1, x2 = _f64(actx, x1, "x1"), _f64(actx, x2, "x2")
    if x1.shape != q.shape or x2.shape != q.shape or out1.shape != q.shape or out2.shape != q.shape:
        raise errors.BindingMismatch("RK operands and outputs must have the shape of the state")
    rk = np.ascontiguousarray(np.asarray(coef, dtype=np.float64).reshape(4))
    _cabi.check(actx.lib.dgb_ns_div_rk_range(disc.handle, q.ptr, T.ptr, gptr, tgptr, x1.ptr, out1.ptr, x2.ptr, out2.ptr,
                                             rk.ctypes.data, op.qfar_host.ctypes.data, op.phys_host.ctypes.data,
                                             int(lo), int(hi), actx._st), "dg_ns_div_rk (range)")
    actx.launch_count += 1

# }}}


# {{{ multi-species reactive Navier-Stokes (multispecies.py): dgb_ms_flux / dgb_ms_div

MS_FUSED_SPECIES = (2, 3, 4)  # the species counts libdgb200 instantiates the kernels for (csrc/dgb_msflux{2,3,4}.cu)


def ms_flux_planes(dim: int, ns: int) -> int:
    return (dim + 1) * (dim + 2 + ns) + 1


def _ms_params(f, qfar, transport, C_):
    mix = getattr(f, "dg_mix", None)
    if mix is None:
        raise errors.BindingMismatch(f"{f.__name__}: the outlined function carries no mixture (f.dg_mix)")
    return _mix_params(mix, qfar, transport, C_)


def _mix_params(mix, qfar, transport, C_):
    m = np.concatenate([[mix.ns], mix.R, mix.cv, mix.h0, [mix.A, mix.Ta, mix.reaction[0], mix.reaction[1]]]).astype(np.float64)
    qf = _host_vec(qfar, C_)
    tr = np.zeros(3) if transport is None else _host_vec(transport, 3)
    return np.ascontiguousarray(m), qf, np.ascontiguousarray(tr)


def _ms_flux(actx, f, q, ghost, Sw, drdx, jac, lift, normals, fscale, vmap_m, vmap_p, bc_kind, qfar, transport):
    dim, ns = f.dg_dim, f.dg_mix.ns
    q = _f64(actx, q, "q")
    G, g, gptr = _ghost_ptr(actx, ghost, (dim + 2 + ns,), q.shape[-1])
    disc = get_disc(actx, dim, q, G, Sw, drdx, lift, normals, fscale, vmap_m, vmap_p, bc_kind, nspecies=ns)
    _bind_jacobian(actx, disc, jac)
    m, qf, tr = _ms_params(f, qfar, transport, dim + 2 + ns)
    out = actx.empty((ms_flux_planes(dim, ns),) + tuple(q.shape[1:]))
    _cabi.check(actx.lib.dgb_ms_flux_range(disc.handle, q.ptr, gptr, out.ptr, qf.ctypes.data, tr.ctypes.data,
                                           m.ctypes.data, 0, -1, actx._st), "dg_ms_flux")
    actx.launch_count += 1
    return out, disc


def _ms_div(actx, f, disc, q, T, ghost, Tghost, jac, facemat, facemat_p, qfar):
    dim, ns = f.dg_dim, f.dg_mix.ns
    q = _f64(actx, q, "q")
    T = _f64(actx, T, "T")
    npl = ms_flux_planes(dim, ns)
    if tuple(T.shape) != (npl,) + tuple(q.shape[1:]):
        raise errors.BindingMismatch(f"flux planes have shape {tuple(T.shape)}, expected {(npl,) + tuple(q.shape[1:])}")
    G, g, gptr = _ghost_ptr(actx, ghost, (dim + 2 + ns,), q.shape[-1])
    TG, tg, tgptr = _ghost_ptr(actx, Tghost, (npl,), q.shape[-1])
    if TG != G:
        raise errors.BindingMismatch("ghost arrays of q and of the flux planes disagree in size")
    _bind_jacobian(actx, disc, jac)
    _check_facemat(disc, facemat, facemat_p)
    m, qf, tr = _ms_params(f, qfar, None, dim + 2 + ns)
    out = actx.empty(q.shape)
    _cabi.check(actx.lib.dgb_ms_div_range(disc.handle, q.ptr, T.ptr, gptr, tgptr, out.ptr, qf.ctypes.data,
                                          tr.ctypes.data, m.ctypes.data, 0, -1, actx._st), "dg_ms_div")
    actx.launch_count += 1
    return out


def _ms_op_disc(actx, op, q, nghost):
    d = op.dcoll
    disc = get_disc(actx, op.dim, q, nghost, d.Sw, d.drdx, d.lift, d.normals, d.fscale, d.vmap_m, d.vmap_p, d.bc_kind,
                    nspecies=op.mix.ns)
    _bind_jacobian(actx, disc, d.jac)
    return disc


def _ms_op_fused(op):
    """The sub-range launches bypass the outlined bodies: refuse when their source no longer matches the kernels."""
    if not (getattr(op._flux, "fused", False) and getattr(op._div, "fused", False)):
        raise errors.BindingMismatch("multi-species sub-range launches need the fused dg_ms_flux / dg_ms_div "
                                     "(operator built with fused=False, or an edited body)")


def ms_flux_range(actx, op, q, ghost, T, lo, hi):
    """``T[:, lo:hi] = dg_ms_flux(q)[:, lo:hi]`` (dgb_ms_flux_range) for a ``MultispeciesOperator``."""
    _ms_op_fused(op)
    q = _f64(actx, q, "q")
    G, g, gptr = _ghost_ptr(actx, ghost, (op.ncomp,), q.shape[-1])
    disc = _ms_op_disc(actx, op, q, G)
    m, qf, tr = _mix_params(op.mix, op.qfar, op.transport, op.ncomp)
    _cabi.check(actx.lib.dgb_ms_flux_range(disc.handle, q.ptr, gptr, T.ptr, qf.ctypes.data, tr.ctypes.data,
                                           m.ctypes.data, int(lo), int(hi), actx._st), "dg_ms_flux (range)")
    actx.launch_count += 1


def ms_div_range(actx, op, q, T, ghost, Tghost, out, lo, hi):
    """``out[:, lo:hi] = dg_ms_div(q, T)[:, lo:hi]`` (dgb_ms_div_range) for a ``MultispeciesOperator``."""
    _ms_op_fused(op)
    q = _f64(actx, q, "q")
    npl = ms_flux_planes(op.dim, op.mix.ns)
    G, g, gptr = _ghost_ptr(actx, ghost, (op.ncomp,), q.shape[-1])
    TG, tg, tgptr = _ghost_ptr(actx, Tghost, (npl,), q.shape[-1])
    disc = _ms_op_disc(actx, op, q, G)
    _check_facemat(disc, op.dcoll.facemat, op.dcoll.facemat_p)
    m, qf, tr = _mix_params(op.mix, op.qfar, None, op.ncomp)
    _cabi.check(actx.lib.dgb_ms_div_range(disc.handle, q.ptr, T.ptr, gptr, tgptr, out.ptr, qf.ctypes.data,
                                          tr.ctypes.data, m.ctypes.data, int(lo), int(hi), actx._st), "dg_ms_div (range)")
    actx.launch_count += 1


def dg_ms_flux(actx, f, q, ghost, Sw, drdx, jac, lift, normals, fscale, vmap_m, vmap_p, bc_kind, qfar, transport):
    return _ms_flux(actx, f, q, ghost, Sw, drdx, jac, lift, normals, fscale, vmap_m, vmap_p, bc_kind, qfar, transport)[0]


def dg_ms_div(actx, f, q, T, ghost, Tghost, Sw, jac, lift, normals, fscale, facemat, facemat_p, vmap_m, vmap_p, bc_kind, qfar):
    dim = f.dg_dim
    G = 0 if ghost is None else ghost.shape[-2]
    disc = actx._discs.get(("nodrdx", dim, G, id(Sw), id(lift), id(normals), id(fscale), id(vmap_m), id(vmap_p), id(bc_kind)))
    if disc is None:
        raise errors.BindingMismatch("dg_ms_div: no discretisation handle for these arrays (call dg_ms_flux first)")
    return _ms_div(actx, f, disc, q, T, ghost, Tghost, jac, facemat, facemat_p, qfar)


def dg_ms_rhs(actx, f, q, Sw, drdx, jac, lift, normals, fscale, facemat, facemat_p, vmap_m, vmap_p, bc_kind, qfar, transport):
    T, disc = _ms_flux(actx, f, q, None, Sw, drdx, jac, lift, normals, fscale, vmap_m, vmap_p, bc_kind, qfar, transport)
    return _ms_div(actx, f, disc, q, T, None, None, jac, facemat, facemat_p, qfar)


def supported(f) -> bool:
    """Whether the fused kernels exist for this outlined function's configuration (else: op by op on the device)."""
    if f.__name__ in ("dg_ms_flux", "dg_ms_div", "dg_ms_rhs"):
        mix = getattr(f, "dg_mix", None)
        return mix is not None and mix.ns in MS_FUSED_SPECIES
    return True

# }}}


FUSED = {"dg_ms_flux": dg_ms_flux, "dg_ms_div": dg_ms_div, "dg_ms_rhs": dg_ms_rhs,
         "dg_ns_flux": dg_ns_flux, "dg_ns_div": dg_ns_div, "dg_ns_div_rk": dg_ns_div_rk, "dg_euler_rhs": dg_euler_rhs, "dg_ns_grad": dg_ns_grad, "dg_ns_rhs": dg_ns_rhs,
         "dg_euler_rhs_rk": dg_euler_rhs_rk, "dg_ns_rhs_rk": dg_ns_rhs_rk}


# {{{ guard of the by-name dispatch: the body must be the one the kernels implement

_FP_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "fused_fingerprints.json")
_FP_CACHE: dict = {}


def fingerprint(f) -> str:
    """SHA-256 over the normalised source (``ast.unparse``: comments and layout do not count) of ``f`` and
    of every Python function it reaches through its closure cells and through global names of its own
    module -- the physics helpers included, so that editing ``inviscid_flux`` or ``_bc_state`` changes the
    fingerprint of every outlined function that uses them."""
    seen, stack = {}, [f]
    while stack:
        g = inspect.unwrap(stack.pop())
        code = getattr(g, "__code__", None)
        if code is None or id(code) in seen:
            continue
        try:
            text = ast.unparse(ast.parse(textwrap.dedent(inspect.getsource(g))))
        except (OSError, TypeError, SyntaxError):
            text = code.co_code.hex() + repr(code.co_consts)
        seen[id(code)] = (g.__qualname__, text)
        names, codes = set(), [code]
        while codes:
            c = codes.pop()
            names.update(c.co_names)
            codes.extend(k for k in c.co_consts if isinstance(k, types.CodeType))
        for n in names:
            v = g.__globals__.get(n)
            if isinstance(v, types.FunctionType) and v.__module__ == g.__module__:
                stack.append(v)
        for cell in g.__closure__ or ():
            try:
                v = cell.cell_contents
            except ValueError:
                continue
            if isinstance(v, types.FunctionType):
                stack.append(v)
    h = hashlib.sha256()
    for name, text in sorted(seen.values()):
        h.update(name.encode() + b"\0" + text.encode() + b"\0")
    return h.hexdigest()


def pinned_fingerprints() -> dict:
    if "pinned" not in _FP_CACHE:
        with open(_FP_PATH) as fh:
            _FP_CACHE["pinned"] = {k: set(v) for k, v in json.load(fh)["functions"].items()}
    return _FP_CACHE["pinned"]


def body_matches(f) -> bool:
    """True if the outlined function ``f`` is (source-identical to) the body the fused kernel named
    ``f.__name__`` was written for (fused_fingerprints.json, regenerated by scripts/make_fingerprints.py)."""
    ok = getattr(f, "_dgb_body_ok", None)           # per function object: closures of one factory share a code object
    if ok is None:
        ok = fingerprint(f) in pinned_fingerprints().get(f.__name__, ())
        try:
            f._dgb_body_ok = ok
        except AttributeError:
            pass
    return ok


def warn_mismatch(name: str) -> None:
    warnings.warn(f"outlined function {name!r} does not match the body its fused B200 kernel implements: "
                  "executing it op by op on the device instead (regenerate fused_fingerprints.json only if the "
                  "kernels were changed accordingly)", RuntimeWarning, stacklevel=3)

# }}}
