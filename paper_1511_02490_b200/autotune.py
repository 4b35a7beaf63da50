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
        h.wgtb_shortlist.restype = ctypes.c_int
        h.wgtb_shortlist.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.POINTER(N.sk_stencil_desc),
                                     ctypes.c_int64, ctypes.c_int64, ctypes.c_int32,
                                     ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int32),
                                     ctypes.POINTER(ctypes.c_int32)]
        h.wgtb_tune_measured.restype = ctypes.c_int
        h.wgtb_tune_measured.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.POINTER(N.sk_stencil_desc),
                                         ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                                         ctypes.c_int64, ctypes.c_int32, ctypes.c_int32,
                                         ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int32),
                                         ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_double),
                                         ctypes.POINTER(ctypes.c_double)]
        h.wgtb_launch_tuned.restype = ctypes.c_int
        h.wgtb_launch_tuned.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.POINTER(N.sk_stencil_desc),
                                        ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                                        ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p,
                                        ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int32),
                                        ctypes.POINTER(ctypes.c_int32)]
        h.wgtb_tuned_refuse.restype = ctypes.c_int
        h.wgtb_tuned_refuse.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.POINTER(N.sk_stencil_desc),
                                        ctypes.c_int64, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32]
        h.wgtb_tuned_reset.restype = None
        h.wgtb_tuned_reset.argtypes = []
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


def shortlist(stencil, width: int, height: int, kernel_json: str | Path,
              model_json: str | Path = RESULTS / "model.json", n: int = 8) -> list[tuple[int, int]]:
    """The model's n best-ranked sizes legal on the current device, best
    first; the first is predict()'s answer (wgtb_shortlist)."""
    wcs, wrs, got = (ctypes.c_int32 * n)(), (ctypes.c_int32 * n)(), ctypes.c_int32()
    rc = lib().wgtb_shortlist(str(model_json).encode(), str(kernel_json).encode(), ctypes.byref(stencil.desc),
                              width, height, n, wcs, wrs, ctypes.byref(got))
    if rc != 0:
        raise RuntimeError(f"wgtb_shortlist: {lib().wgtb_last_error().decode()}")
    return [(wcs[i], wrs[i]) for i in range(got.value)]


def tune_measured(stencil, inp, out, kernel_json: str | Path, model_json: str | Path = RESULTS / "model.json",
                  n: int = 8, samples: int = 5) -> dict:
    """Prediction refined by measurement (wgtb_tune_measured): the model's
    n-size shortlist timed on inp -> out (median of `samples` flushed
    passes each); {'wc', 'wr', 'timed', 'best_ms', 'ms'} of the fastest."""
    stencil._check_device(inp, out)
    h, w = out.shape
    wc, wr, timed = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
    best, ms = ctypes.c_double(), ctypes.c_double()
    rc = lib().wgtb_tune_measured(str(model_json).encode(), str(kernel_json).encode(), ctypes.byref(stencil.desc),
                                  inp.data_ptr(), out.data_ptr(), w, h, inp.stride(0), n, samples,
                                  ctypes.byref(wc), ctypes.byref(wr), ctypes.byref(timed), ctypes.byref(best),
                                  ctypes.byref(ms))
    if rc != 0:
        raise RuntimeError(f"wgtb_tune_measured: {lib().wgtb_last_error().decode()}")
    return {"wc": wc.value, "wr": wr.value, "timed": timed.value, "best_ms": best.value, "ms": ms.value}


class Tuned:
    """Online-tuned launches of `stencil` (wgtb_launch_tuned): the model
    proposes the workgroup size once per (grid, device) session and
    re-proposes when a launch is refused - the refused size is never proposed
    again in the session (reference serve.cpp:123-164)."""

    def __init__(self, stencil, kernel_json: str | Path, model_json: str | Path = RESULTS / "model.json"):
        self.stencil = stencil
        self.kernel_json = str(kernel_json).encode()
        self.model_json = str(model_json).encode()
        self.last = None  # (wc, wr, proposals) of the last launch

    def __call__(self, inp, out, stream=None) -> tuple[int, int]:
        import torch

        self.stencil._check_device(inp, out)
        h, w = out.shape
        s = (stream or torch.cuda.current_stream(inp.device)).cuda_stream
        wc, wr, props = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
        rc = lib().wgtb_launch_tuned(self.model_json, self.kernel_json, ctypes.byref(self.stencil.desc),
                                     inp.data_ptr(), out.data_ptr(), w, h, inp.stride(0), out.stride(0),
                                     s or None, ctypes.byref(wc), ctypes.byref(wr), ctypes.byref(props))
        if rc != 0:
            raise RuntimeError(f"wgtb_launch_tuned: {lib().wgtb_last_error().decode()}")
        self.last = (wc.value, wr.value, props.value)
        return wc.value, wr.value

    def refuse(self, width: int, height: int, wc: int, wr: int) -> None:
        """External refusal feedback for the (width x height) session."""
        rc = lib().wgtb_tuned_refuse(self.model_json, self.kernel_json, ctypes.byref(self.stencil.desc),
                                     width, height, wc, wr)
        if rc != 0:
            raise RuntimeError(f"wgtb_tuned_refuse: {lib().wgtb_last_error().decode()}")

    @staticmethod
    def reset() -> None:
        lib().wgtb_tuned_reset()
