"""ctypes binding of the C-ABI in include/sk_stencil.h.

The shared library is built in-tree (paper_1511_02490_b200/lib/libsk_stencil.so,
see __graft_entry__.build()).  There is no fallback: if the library is missing
or fails to load, every entry point raises.
"""
from __future__ import annotations

import ctypes
import os
import re
from pathlib import Path

PKG_DIR = Path(__file__).resolve().parent
REPO_ROOT = PKG_DIR.parent
LIB_PATH = PKG_DIR / "lib" / "libsk_stencil.so"
HEADER_PATH = REPO_ROOT / "include" / "sk_stencil.h"

# sk_status (include/sk_stencil.h)
SK_OK, SK_OVERSIZED, SK_REFUSED, SK_EINVAL, SK_ECUDA, SK_ENOTSUP = range(6)
STATUS_NAMES = {0: "OK", 1: "OVERSIZED", 2: "REFUSED", 3: "EINVAL", 4: "ECUDA", 5: "ENOTSUP"}

# sk_dtype, in reference ElementType order (scenario.hpp:14)
SK_INT32, SK_FLOAT32, SK_FLOAT64 = 0, 1, 2
DTYPE_NAMES = {SK_INT32: "INT32", SK_FLOAT32: "FLOAT32", SK_FLOAT64: "FLOAT64"}
DTYPE_SIZE = {SK_INT32: 4, SK_FLOAT32: 4, SK_FLOAT64: 8}

SK_BORDER_PAD, SK_BORDER_NEAREST = 0, 1
SK_LOAD_AUTO, SK_LOAD_TMA, SK_LOAD_EXPLICIT, SK_LOAD_BITPLANE, SK_LOAD_STRIPS, SK_LOAD_VECTOR = 0, 1, 2, 3, 4, 5

# sk_op
OPS = {
    "five_point": 0,
    "heat": 1,
    "gol": 2,
    "boxmean": 3,
    "gaussian": 4,
    "sobel": 5,
    "nms": 6,
    "threshold": 7,
    "synthetic": 8,
}


class sk_stencil_desc(ctypes.Structure):
    _fields_ = [
        ("op", ctypes.c_int32),
        ("dtype", ctypes.c_int32),
        ("north", ctypes.c_int32),
        ("south", ctypes.c_int32),
        ("east", ctypes.c_int32),
        ("west", ctypes.c_int32),
        ("border_mode", ctypes.c_int32),
        ("pad_value", ctypes.c_double),
        ("complexity", ctypes.c_int32),
        ("instructions", ctypes.c_int32),
        ("load_path", ctypes.c_int32),
        ("cells_per_thread", ctypes.c_int32),
        ("fused_iterations", ctypes.c_int32),
    ]


class sk_device_props(ctypes.Structure):
    _fields_ = [
        ("name", ctypes.c_char * 128),
        ("compute_units", ctypes.c_int32),
        ("frequency_mhz", ctypes.c_int32),
        ("local_mem_kb", ctypes.c_int32),
        ("global_cache_kb", ctypes.c_int32),
        ("global_mem_mb", ctypes.c_int32),
        ("device_max_wgsize", ctypes.c_int32),
        ("simd_width", ctypes.c_int32),
        ("cc_major", ctypes.c_int32),
        ("cc_minor", ctypes.c_int32),
        ("mem_clock_mhz", ctypes.c_int32),
        ("mem_bus_width", ctypes.c_int32),
    ]


class NativeError(RuntimeError):
    """A non-OK status from the C-ABI (carries the code and sk_last_error())."""

    def __init__(self, code: int, where: str, message: str):
        super().__init__(f"{where}: {STATUS_NAMES.get(code, code)}: {message}")
        self.code = code


class sk_ipc_handle(ctypes.Structure):
    _fields_ = [("handle", ctypes.c_ubyte * 64), ("offset", ctypes.c_int64)]


class sk_halo_peers(ctypes.Structure):
    _fields_ = [
        ("north_a", ctypes.c_void_p),
        ("north_b", ctypes.c_void_p),
        ("south_a", ctypes.c_void_p),
        ("south_b", ctypes.c_void_p),
        ("north_control", ctypes.c_void_p),
        ("south_control", ctypes.c_void_p),
        ("north_rows", ctypes.c_int64),
    ]


SK_HALO_CONTROL_BYTES = 64

_lib = None

_i32, _i64, _vp = ctypes.c_int32, ctypes.c_int64, ctypes.c_void_p
_desc_p = ctypes.POINTER(sk_stencil_desc)

_PROTOTYPES = {
    "sk_stencil_launch": (_i32, [_desc_p, _vp, _vp, _i64, _i64, _i64, _i64, _i64, _i64, _i32, _i32, _vp]),
    "sk_stencil_launch_custom": (_i32, [_desc_p, _vp, _vp, _vp, _i64, _i64, _i64, _i64, _i64, _i64,
                                        _i32, _i32, _vp]),
    "sk_stencil_iterate": (_i32, [_desc_p, _vp, _vp, _i64, _i64, _i64, _i32, _i32, _i32, _vp,
                                  ctypes.POINTER(_i32)]),
    "sk_stencil_probe": (_i32, [_desc_p, _i64, _i64, _i32, _i32, ctypes.POINTER(_i32),
                                ctypes.POINTER(_i64), ctypes.POINTER(_i32)]),
    "sk_kernel_max_wgsize": (_i32, [_desc_p, ctypes.POINTER(_i32)]),
    "sk_stencil_time": (_i32, [_desc_p, _vp, _vp, _i64, _i64, _i64, _i32, _i32, _i32, _i32, _i32,
                               ctypes.POINTER(ctypes.c_double)]),
    "sk_copy_time": (_i32, [_vp, _vp, _i64, _i32, _i32, _i32, _i32, ctypes.POINTER(ctypes.c_double)]),
    "sk_stencil_run_host": (_i32, [_desc_p, _vp, _vp, _i64, _i64, _i32, _i32, _i32]),
    "sk_stencil_submit_host": (_i32, [_desc_p, _vp, _vp, _i64, _i64, _i32, _i32, _i32,
                                      ctypes.POINTER(_i64)]),
    "sk_stencil_wait_host": (_i32, [_i64]),
    "sk_device_features": (_i32, [_i32, ctypes.POINTER(sk_device_props)]),
    "sk_fill_host": (_i32, [_i32, _i32, ctypes.c_uint64, _vp, _i64]),
    "sk_buffers_equal": (_i32, [_vp, _vp, _i64, ctypes.POINTER(_i32)]),
    "sk_ipc_export": (_i32, [_vp, ctypes.POINTER(sk_ipc_handle)]),
    "sk_ipc_import": (_i32, [ctypes.POINTER(sk_ipc_handle), ctypes.POINTER(_vp)]),
    "sk_ipc_close": (_i32, [_vp]),
    "sk_stencil_iterate_nccl": (_i32, [_desc_p, _vp, _vp, _i64, _i64, _i64, _i32, _i32, _i32, _vp,
                                       _i32, _i32, _vp, ctypes.POINTER(ctypes.c_int32)]),
    "sk_stencil_iterate_peer": (_i32, [_desc_p, _vp, _vp, _i64, _i64, _i64, _i32, _i32, _i32,
                                       ctypes.POINTER(sk_halo_peers), _vp, ctypes.POINTER(_i64),
                                       _vp, ctypes.POINTER(_i32)]),
    "sk_last_error": (ctypes.c_char_p, []),
    "sk_version": (ctypes.c_char_p, []),
}


def header_symbols() -> list[str]:
    """Entry points declared in include/sk_stencil.h."""
    text = HEADER_PATH.read_text()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(sk_\w+)\s*\(", text, re.M)))


def lib() -> ctypes.CDLL:
    """Load the native library (raises if it is missing — no fallback)."""
    global _lib
    if _lib is None:
        path = Path(os.environ.get("SK_STENCIL_LIB", str(LIB_PATH)))
        if not path.exists():
            raise ImportError(
                f"native stencil library not found at {path}; run __graft_entry__.build()")
        handle = ctypes.CDLL(str(path))
        for name, (res, args) in _PROTOTYPES.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


def last_error() -> str:
    return lib().sk_last_error().decode()


def check(code: int, where: str) -> int:
    if code != SK_OK:
        raise NativeError(code, where, last_error())
    return code
