"""paper_1511_02490_b200 — B200-native SkelCL stencil executor + workgroup-size autotuner.

The hot path (a Stencil pass at a runtime wc x wr block) is hand-written
sm_100a CUDA behind the C-ABI in include/sk_stencil.h; the autotuner (the
reference's wgtune: space, features, learn, tuner, bench) is native C++ in
csrc/host.  This package is the Python mirror used by tests and bench.py.
"""
from ._native import NativeError, lib  # noqa: F401
from .stencil import (IllegalWorkgroupSize, RefusedParameter, Stencil,  # noqa: F401
                      copy_time, device_features, fill_host)

__all__ = ["Stencil", "RefusedParameter", "IllegalWorkgroupSize", "NativeError", "lib",
           "copy_time", "device_features", "fill_host"]
