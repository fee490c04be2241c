"""Reference-side binding of libdgb200.so: what a `laze` maintainer adds next to `laze/backend.py`.

`run_call_step_b200(function_name, arrays)` is a drop-in for the `CallStep` branch of the reference's
interpreter `run_ir` (/root/reference/pkg/src/laze/backend.py:90-96) for the outlined DG functions of the
default Navier-Stokes arrangement, `dg_ns_flux` and `dg_ns_div`: `arrays` maps the parameter names
`_p0, _p1, ...` (/root/reference/pkg/src/laze/frontend.py:501) to the NumPy arrays the interpreter has
bound, the return value maps result names to NumPy arrays (a single result is called "out",
frontend.py:575).  Nothing but `ctypes`, NumPy and the C ABI of include/dgb200.h is used -- no torch,
no other module of this repository; device memory comes from the library's own allocator.

tests/test_gpu_parity.py::test_integration_stub_executes runs this file against the oracle.
"""
import ctypes as C
import itertools
import os

import numpy as np

_LIB_PATH = os.environ.get("DGB_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "..",
                                                      "paper_2512_17101_b200", "libdgb200.so")
_lib = C.CDLL(_LIB_PATH)
_lib.dgb_last_error.restype = C.c_char_p
_VP, _I64 = C.c_void_p, C.c_int64
_lib.dgb_malloc.argtypes = [C.POINTER(_VP), C.c_size_t]
_lib.dgb_free.argtypes = [_VP]
_lib.dgb_memcpy_h2d.argtypes = [_VP, _VP, C.c_size_t, _VP]
_lib.dgb_memcpy_d2h.argtypes = [_VP, _VP, C.c_size_t, _VP]
_lib.dgb_stream_sync.argtypes = [_VP]
_lib.dgb_disc_create.argtypes = [C.POINTER(_VP), C.c_int, C.c_int, _I64, _I64] + [_VP] * 11
_lib.dgb_disc_destroy.argtypes = [_VP]
_lib.dgb_disc_set_jacobian.argtypes = [_VP, _VP, _VP]
_lib.dgb_ns_flux.argtypes = [_VP] * 7
_lib.dgb_ns_div.argtypes = [_VP] * 9

# status -> exception class name of laze/errors.py (include/dgb200.h: dgb_status)
_ERR = {2: "ShapeMismatch", 3: "OutOfBoundsIndex", 4: "BindingMismatch", 5: "DTypeMismatch"}


def _check(status):
    if status:
        msg = _lib.dgb_last_error().decode()
        try:
            from laze import errors                      # on the reference side: its own exception classes
            raise getattr(errors, _ERR.get(status, "LazeError"))(msg)
        except ImportError:
            raise RuntimeError(f"{_ERR.get(status, 'LazeError')}: {msg}") from None


class _Dev:
    """A device buffer owned by the executor."""

    def __init__(self, host=None, shape=None):
        if host is not None:
            host = np.ascontiguousarray(host)
            shape = host.shape
        self.shape = tuple(shape)
        self.nbytes = int(np.prod(self.shape, dtype=np.int64)) * 8
        self.ptr = _VP()
        _check(_lib.dgb_malloc(C.byref(self.ptr), self.nbytes))
        if host is not None:
            assert host.dtype.itemsize == 8
            _check(_lib.dgb_memcpy_h2d(self.ptr, host.ctypes.data, host.nbytes, None))
            _check(_lib.dgb_stream_sync(None))           # pageable source: copy done before `host` may die

    def to_host(self):
        out = np.empty(self.shape, np.float64)
        _check(_lib.dgb_memcpy_d2h(out.ctypes.data, self.ptr, out.nbytes, None))
        _check(_lib.dgb_stream_sync(None))
        return out

    def __del__(self):
        try:
            _lib.dgb_free(self.ptr)
        except Exception:
            pass


_ORDER = {(2, 3): 1, (2, 6): 2, (2, 10): 3, (2, 15): 4, (3, 4): 1, (3, 10): 2, (3, 20): 3, (3, 35): 4}
_HANDLES = {}      # per mesh: creating the handle validates and compresses the int64 face maps once


def _face_tables(dim, order, vmap_m, Np):
    """(Nf, Nfp) volume-node numbers of the face nodes, read off the application's own `vmap_m` of element 0,
    and the (dim!, Nfp) position permutations of a face's nodes under permutations of its vertices, which
    depend on the element family only (paper_2512_17101_b200.dg.simplex.SimplexElement.face_perms)."""
    from paper_2512_17101_b200.dg.simplex import simplex_element    # element tables: setup-time NumPy only
    el = simplex_element(dim, order)
    Nf, Nfp = el.Nf, el.Nfp
    fn = np.ascontiguousarray(vmap_m.reshape(-1)[:Nf * Nfp].reshape(Nf, Nfp) % Np, dtype=np.int64)
    assert np.array_equal(fn, el.face_nodes)
    assert el.face_perms.shape == (len(list(itertools.permutations(range(dim)))), Nfp)
    return fn, np.ascontiguousarray(el.face_perms, dtype=np.int64)


def _handle(q, Sw, drdx, jac, lift, nrm, fsc, vm, vp, bc):
    key = (vm.ctypes.data, vp.ctypes.data, q.shape)
    h = _HANDLES.get(key)
    if h is None:
        C_, E, Np = q.shape
        dim = C_ - 2
        order = _ORDER[(dim, Np)]
        fn, fp = _face_tables(dim, order, vm, Np)
        dev = {k: _Dev(v) for k, v in dict(drdx=drdx, nrm=nrm, fsc=fsc, vm=vm, vp=vp, bc=bc, jac=jac).items()}
        disc = _VP()
        Sw, lift = np.ascontiguousarray(Sw), np.ascontiguousarray(lift)
        _check(_lib.dgb_disc_create(C.byref(disc), dim, order, E, 0, Sw.ctypes.data, lift.ctypes.data,
                                    fn.ctypes.data, fp.ctypes.data, dev["drdx"].ptr, dev["nrm"].ptr, dev["fsc"].ptr,
                                    dev["vm"].ptr, dev["vp"].ptr, dev["bc"].ptr, None))
        _check(_lib.dgb_disc_set_jacobian(disc, dev["jac"].ptr, None))
        h = _HANDLES[key] = (disc, dev)
    return h[0]


def run_call_step_b200(function_name, arrays):
    p = [arrays[f"_p{k}"] for k in range(len(arrays))]
    if function_name == "dg_ns_flux":
        q, Sw, drdx, jac, lift, nrm, fsc, vm, vp, bc, qfar, phys = p
        disc = _handle(q, Sw, drdx, jac, lift, nrm, fsc, vm, vp, bc)
        dq = _Dev(q)
        T = _Dev(shape=((q.shape[0] - 1) * q.shape[0] + 1,) + q.shape[1:])      # (dim+1)*C + 1 planes, C = dim + 2
        qf, ph = np.ascontiguousarray(qfar.reshape(-1)), np.ascontiguousarray(phys.reshape(-1))
        _check(_lib.dgb_ns_flux(disc, dq.ptr, None, T.ptr, qf.ctypes.data, ph.ctypes.data, None))
        return {"out": T.to_host()}
    if function_name == "dg_ns_div":
        q, T, Sw, jac, lift, nrm, fsc, facemat, facemat_p, vm, vp, bc, qfar, phys = p
        key = (vm.ctypes.data, vp.ctypes.data, q.shape)
        if key not in _HANDLES:
            raise RuntimeError("dg_ns_div before dg_ns_flux on this mesh")
        disc = _HANDLES[key][0]
        dq, dT, out = _Dev(q), _Dev(T), _Dev(shape=q.shape)
        qf, ph = np.ascontiguousarray(qfar.reshape(-1)), np.ascontiguousarray(phys.reshape(-1))
        _check(_lib.dgb_ns_div(disc, dq.ptr, dT.ptr, None, None, out.ptr, qf.ctypes.data, ph.ctypes.data, None))
        return {"out": out.to_host()}
    raise KeyError(function_name)


def close():
    for disc, _ in _HANDLES.values():
        _lib.dgb_disc_destroy(disc)
    _HANDLES.clear()
