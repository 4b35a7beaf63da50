"""Python mirror of the in-process autotuner call (include/wgtb_c.h):
ask the trained model for a workgroup size, with refusals probed live on the
device (the paper's SkelCL <-> daemon loop)."""
from __future__ import annotations

import ctypes
from pathlib import Path

from . import _native as N

LIB = N.PKG_DIR / "lib" / "libwgtb.so"
RESULTS = N.REPO_ROOT / "results" / "b200"
_lib = None


def lib():
    global _lib
    if _lib is None:
        N.lib()  # libsk_stencil first (libwgtb links against it)
        if not LIB.exists():
            raise ImportError(f"{LIB} not built; run __graft_entry__.build()")
        h = ctypes.CDLL(str(LIB))
        h.wgtb_predict.restype = ctypes.c_int
        h.wgtb_predict.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.POINTER(N.sk_stencil_desc),
                                   ctypes.c_int64, ctypes.c_int64, ctypes.POINTER(ctypes.c_int32),
                                   ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int32),
                                   ctypes.POINTER(ctypes.c_double)]
        h.wgtb_last_error.restype = ctypes.c_char_p
        _lib = h
    return _lib


def predict(stencil, width: int, height: int, kernel_json: str | Path,
            model_json: str | Path = RESULTS / "model.json") -> dict:
    """{'wc', 'wr', 'probes', 'ms'} for `stencil` on a width x height grid."""
    wc, wr, probes, ms = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32(), ctypes.c_double()
    rc = lib().wgtb_predict(str(model_json).encode(), str(kernel_json).encode(),
                            ctypes.byref(stencil.desc), width, height, ctypes.byref(wc),
                            ctypes.byref(wr), ctypes.byref(probes), ctypes.byref(ms))
    if rc != 0:
        raise RuntimeError(f"wgtb_predict: {lib().wgtb_last_error().decode()}")
    return {"wc": wc.value, "wr": wr.value, "probes": probes.value, "ms": ms.value}
