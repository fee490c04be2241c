"""ctypes binding of ``libdgb200.so`` (C ABI declared in include/dgb200.h).

The library is built in-tree by ``__graft_entry__.build()`` / ``csrc/build.py``.  If it is
missing this module raises ``ExtensionMissing`` -- the product has no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os

from . import errors

_LIB = None
LIB_PATH = os.environ.get("DGB_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "libdgb200.so")

# every symbol include/dgb200.h declares (tests/test_cabi_symbols.py checks the two stay in sync)
SYMBOLS = [
    "dgb_last_error", "dgb_version", "dgb_malloc", "dgb_free", "dgb_host_alloc", "dgb_host_free",
    "dgb_memcpy_h2d", "dgb_memcpy_d2h", "dgb_memcpy_d2d", "dgb_stream_sync",
    "dgb_disc_create", "dgb_disc_destroy", "dgb_disc_expand_maps", "dgb_debug_phase_cycles",
    "dgb_euler_rhs", "dgb_ns_grad", "dgb_ns_rhs", "dgb_euler_rhs_rk", "dgb_ns_rhs_rk",
    "dgb_disc_set_jacobian", "dgb_ns_flux", "dgb_ns_div", "dgb_ns_div_rk",
    "dgb_euler_rhs_range", "dgb_ns_flux_range", "dgb_ns_div_range", "dgb_ns_div_rk_range", "dgb_ms_flux_range", "dgb_ms_div_range", "dgb_ms_div_rk",
    "dgb_pack_elements", "dgb_pack_elements_to", "dgb_ipc_alloc", "dgb_ipc_open", "dgb_ipc_close",
    "dgb_flag_signal", "dgb_flag_wait",
    "dgb_ew_binary", "dgb_ew_unary", "dgb_ew_where", "dgb_copy_strided", "dgb_copy_scatter", "dgb_take", "dgb_take_deferred",
    "dgb_einsum", "dgb_ew_program", "dgb_set_sm_reserve",
]

DGB_OK, DGB_ERR_CUDA, DGB_ERR_INVALID, DGB_ERR_OUT_OF_BOUNDS, DGB_ERR_BAD_MAP, DGB_ERR_DTYPE = range(6)

_STATUS_TO_EXC = {
    DGB_ERR_CUDA: errors.LazeError,
    DGB_ERR_INVALID: errors.ShapeMismatch,
    DGB_ERR_OUT_OF_BOUNDS: errors.OutOfBoundsIndex,
    DGB_ERR_BAD_MAP: errors.BindingMismatch,
    DGB_ERR_DTYPE: errors.DTypeMismatch,
}

BINOPS = {name: k for k, name in enumerate(
    ["add", "sub", "mul", "truediv", "floordiv", "mod", "pow", "min", "max", "lt", "le", "gt", "ge", "eq", "ne"])}
UNOPS = {name: k for k, name in enumerate(["neg", "abs", "sqrt", "exp", "log"])}


# dgb_ew_program (include/dgb200.h)
EW_MAX_INS, EW_MAX_REGS, EW_MAX_LEAVES, EW_MAX_OUTS, EW_MAX_CONSTS = 96, 32, 12, 4, 24
EW_LOAD, EW_CONST, EW_BINARY, EW_UNARY, EW_WHERE = range(5)


class EwIns(C.Structure):
    _fields_ = [(n, C.c_uint8) for n in ("kind", "op", "dst", "a", "b", "c", "adt", "bdt", "cdt", "odt", "fcomp", "pad_")]


class EwLeaf(C.Structure):
    _fields_ = [("dev", C.c_void_p), ("dtype", C.c_int32), ("mode", C.c_int32), ("stride", C.c_int64 * 8)]


class EwOut(C.Structure):
    _fields_ = [("dev", C.c_void_p), ("dtype", C.c_int32), ("reg", C.c_int32)]


class EwProg(C.Structure):
    _fields_ = [("nins", C.c_int32), ("nleaves", C.c_int32), ("nouts", C.c_int32), ("rank", C.c_int32),
                ("need_index", C.c_int32), ("pad_", C.c_int32), ("total", C.c_int64), ("ext", C.c_int64 * 8),
                ("consts", C.c_uint64 * EW_MAX_CONSTS), ("leaf", EwLeaf * EW_MAX_LEAVES), ("out", EwOut * EW_MAX_OUTS),
                ("ins", EwIns * EW_MAX_INS)]


def load():
    """Load the shared library once; raise ``ExtensionMissing`` if it is not there."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(LIB_PATH):
        raise errors.ExtensionMissing(
            f"{LIB_PATH} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(nvcc, sm_100a).  There is no CPU fallback.")
    try:
        lib = C.CDLL(LIB_PATH)
    except OSError as exc:  # pragma: no cover
        raise errors.ExtensionMissing(f"cannot load {LIB_PATH}: {exc}") from exc
    missing = [s for s in SYMBOLS if not hasattr(lib, s)]
    if missing:
        raise errors.ExtensionMissing(f"{LIB_PATH} lacks symbols {missing}; rebuild it")
    lib.dgb_last_error.restype = C.c_char_p
    vp, i64, dp = C.c_void_p, C.c_int64, C.c_void_p
    lib.dgb_malloc.argtypes = [C.POINTER(C.c_void_p), C.c_size_t]
    lib.dgb_free.argtypes = [vp]
    lib.dgb_host_alloc.argtypes = [C.POINTER(C.c_void_p), C.c_size_t]
    lib.dgb_host_free.argtypes = [vp]
    for name in ("dgb_memcpy_h2d", "dgb_memcpy_d2h", "dgb_memcpy_d2d"):
        getattr(lib, name).argtypes = [vp, vp, C.c_size_t, vp]
    lib.dgb_stream_sync.argtypes = [vp]
    lib.dgb_disc_create.argtypes = [C.POINTER(C.c_void_p), C.c_int, C.c_int, i64, i64,
                                    vp, vp, vp, vp, dp, dp, dp, dp, dp, dp, vp]
    lib.dgb_disc_destroy.argtypes = [vp]
    lib.dgb_disc_expand_maps.argtypes = [vp, dp, dp, vp]
    lib.dgb_debug_phase_cycles.argtypes = [vp, vp]
    lib.dgb_euler_rhs.argtypes = [vp, dp, dp, dp, vp, vp, vp]
    lib.dgb_ns_grad.argtypes = [vp, dp, dp, dp, vp, vp]
    lib.dgb_ns_rhs.argtypes = [vp, dp, dp, dp, dp, dp, vp, vp, vp]
    lib.dgb_euler_rhs_rk.argtypes = [vp, dp, dp, dp, dp, dp, dp, vp, vp, vp, vp]
    lib.dgb_ns_rhs_rk.argtypes = [vp, dp, dp, dp, dp, dp, dp, dp, dp, vp, vp, vp, vp]
    lib.dgb_disc_set_jacobian.argtypes = [vp, dp, vp]
    lib.dgb_ns_flux.argtypes = [vp, dp, dp, dp, vp, vp, vp]
    lib.dgb_ns_div.argtypes = [vp, dp, dp, dp, dp, dp, vp, vp, vp]
    lib.dgb_ns_div_rk.argtypes = [vp, dp, dp, dp, dp, dp, dp, dp, dp, vp, vp, vp, vp]
    lib.dgb_euler_rhs_range.argtypes = [vp, dp, dp, dp, vp, vp, i64, i64, vp]
    lib.dgb_ns_flux_range.argtypes = [vp, dp, dp, dp, vp, vp, i64, i64, vp]
    lib.dgb_ns_div_range.argtypes = [vp, dp, dp, dp, dp, dp, vp, vp, i64, i64, vp]
    lib.dgb_ns_div_rk_range.argtypes = [vp, dp, dp, dp, dp, dp, dp, dp, dp, vp, vp, vp, i64, i64, vp]
    lib.dgb_ms_flux_range.argtypes = [vp, dp, dp, dp, vp, vp, vp, i64, i64, vp]
    lib.dgb_ms_div_range.argtypes = [vp, dp, dp, dp, dp, dp, vp, vp, vp, i64, i64, vp]
    lib.dgb_ms_div_rk.argtypes = [vp, dp, dp, dp, dp, dp, dp, dp, dp, vp, vp, vp, vp, vp]
    lib.dgb_pack_elements.argtypes = [dp, dp, dp, i64, i64, i64, i64, vp]
    lib.dgb_pack_elements_to.argtypes = [dp, i64, i64, dp, dp, i64, i64, i64, i64, vp]
    lib.dgb_ipc_alloc.argtypes = [C.POINTER(C.c_void_p), C.c_size_t, vp]
    lib.dgb_ipc_open.argtypes = [C.POINTER(C.c_void_p), vp]
    lib.dgb_ipc_close.argtypes = [vp]
    lib.dgb_flag_signal.argtypes = [vp, C.c_uint64, vp]
    lib.dgb_flag_wait.argtypes = [vp, C.c_uint64, vp]
    lib.dgb_ew_binary.argtypes = [C.c_int, dp, C.c_int, dp, C.c_int, vp, dp, C.c_int, vp, C.c_int, vp, vp]
    lib.dgb_ew_unary.argtypes = [C.c_int, dp, C.c_int, dp, C.c_int, i64, vp]
    lib.dgb_ew_where.argtypes = [dp, C.c_int, dp, C.c_int, vp, dp, C.c_int, vp, dp, C.c_int, vp, C.c_int, vp, vp]
    lib.dgb_copy_strided.argtypes = [dp, C.c_int, dp, C.c_int, vp, C.c_int, vp, vp]
    lib.dgb_copy_scatter.argtypes = [dp, C.c_int, vp, dp, C.c_int, vp, C.c_int, vp, vp]
    lib.dgb_take.argtypes = [dp, dp, C.c_int, dp, i64, i64, i64, i64, vp]
    lib.dgb_take_deferred.argtypes = [dp, dp, C.c_int, dp, i64, i64, i64, i64, vp, vp]
    lib.dgb_einsum.argtypes = [dp, C.c_int, vp, vp, C.c_int, C.c_int, vp, vp]
    lib.dgb_set_sm_reserve.argtypes = [C.c_int]
    lib.dgb_ew_program.argtypes = [C.POINTER(EwProg), vp]
    _LIB = lib
    return lib


def check(status: int, what: str = "") -> None:
    if status == DGB_OK:
        return
    msg = load().dgb_last_error().decode() or f"status {status}"
    raise _STATUS_TO_EXC.get(status, errors.LazeError)(f"{what}: {msg}" if what else msg)


def i64_array(values):
    return (C.c_int64 * len(values))(*[int(v) for v in values])
