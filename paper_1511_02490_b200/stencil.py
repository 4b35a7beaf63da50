"""Python mirror of the C++ ``skelcl::Stencil<T>`` host API (include/wgtb/stencil.hpp).

A Stencil is the SkelCL pattern of PAPER.md:87-117: a customising function
(``op``), a rectangular N/S/E/W border region, a border mode (pad value or
nearest cell) and a runtime workgroup size ``wc x wr`` chosen per call.
All work goes through the C-ABI (include/sk_stencil.h); there is no CPU path.

Device buffers are torch CUDA tensors (torch is plumbing only: memory and
streams).  Row pitch is ``tensor.stride(0)``.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

from . import _native as N

# Reference kernel names (synthgen.cpp:82-96, Table 2) -> ops.
REFERENCE_KERNEL_OPS = {
    "gaussian": "gaussian",
    "gol": "gol",
    "he": "heat",
    "nms": "nms",
    "sobel": "sobel",
    "threshold": "threshold",
}

_TORCH_DTYPE_NAMES = {"int32": N.SK_INT32, "float32": N.SK_FLOAT32, "float64": N.SK_FLOAT64}


def dtype_code(dtype) -> int:
    """Accepts sk codes, reference names ("INT32"), numpy or torch dtypes."""
    if isinstance(dtype, int):
        return dtype
    s = str(dtype).split(".")[-1].lower()
    if s in _TORCH_DTYPE_NAMES:
        return _TORCH_DTYPE_NAMES[s]
    raise ValueError(f"unsupported element type {dtype!r}")


class RefusedParameter(RuntimeError):
    """The device refused (wc, wr) (reference errors.hpp:52-63)."""

    def __init__(self, message: str, w_c: int, w_r: int):
        super().__init__(message)
        self.w_c, self.w_r = w_c, w_r


class IllegalWorkgroupSize(RuntimeError):
    """wc*wr exceeds the effective maximum (reference errors.hpp:27)."""


@dataclass
class Stencil:
    op: str
    dtype: object = "float32"
    north: int = 1
    south: int = 1
    east: int = 1
    west: int = 1
    border: str = "pad"          # "pad" | "nearest"
    pad_value: float = 0.0
    complexity: int = 0          # synthetic kernels only
    instructions: int = 100      # synthetic kernels only
    load_path: str = "auto"      # "auto" | "tma" | "explicit" | "bitplane" (gol)
                                 # | "strips" (five_point / heat, unit borders)
                                 # | "vector" (16-B vector work-items: five_point,
                                 #   heat, gol, sobel, nms unit borders; boxmean 5,1,3,0)
    cells_per_thread: int = 0    # K cells per work-item; 0 = auto
    fused_iterations: int = 0    # temporal blocking: generations per launch
                                 # (0/1, 2, 4; gol on the bit-plane path: 1..128;
                                 # five_point / heat on the strip path: 1..32)
    _desc: N.sk_stencil_desc = field(init=False, repr=False)

    def __post_init__(self):
        if self.op not in N.OPS:
            raise ValueError(f"unknown op {self.op!r}")
        self._desc = N.sk_stencil_desc(
            op=N.OPS[self.op], dtype=dtype_code(self.dtype), north=self.north, south=self.south,
            east=self.east, west=self.west,
            border_mode=N.SK_BORDER_NEAREST if self.border == "nearest" else N.SK_BORDER_PAD,
            pad_value=float(self.pad_value), complexity=int(self.complexity),
            instructions=int(self.instructions),
            load_path={"auto": N.SK_LOAD_AUTO, "tma": N.SK_LOAD_TMA,
                       "explicit": N.SK_LOAD_EXPLICIT,
                       "bitplane": N.SK_LOAD_BITPLANE,
                       "strips": N.SK_LOAD_STRIPS,
                       "vector": N.SK_LOAD_VECTOR}[self.load_path],
            cells_per_thread=int(self.cells_per_thread),
            fused_iterations=int(self.fused_iterations))

    # -- construction from reference descriptors ---------------------------
    @classmethod
    def from_kernel(cls, name: str, north: int, south: int, east: int, west: int,
                    dtype="float32", complexity: int = 0, instructions: int = 100,
                    border: str = "pad", pad_value: float = 0.0, **kw) -> "Stencil":
        """Executable stencil for a reference KernelDescriptor (scenario.hpp:46-56)."""
        if name.startswith("synthetic-"):
            op = "synthetic"
        elif name in REFERENCE_KERNEL_OPS:
            op = REFERENCE_KERNEL_OPS[name]
        elif name in N.OPS:
            op = name
        else:
            raise ValueError(f"no executable functor for kernel {name!r}")
        return cls(op=op, dtype=dtype, north=north, south=south, east=east, west=west,
                   border=border, pad_value=pad_value, complexity=complexity,
                   instructions=instructions, **kw)

    @property
    def desc(self) -> N.sk_stencil_desc:
        return self._desc

    @property
    def dtype_code(self) -> int:
        return self._desc.dtype

    # -- execution -----------------------------------------------------------
    def _raise(self, code: int, where: str, wc: int, wr: int):
        msg = f"{where}: {N.last_error()}"
        if code == N.SK_REFUSED:
            raise RefusedParameter(msg, wc, wr)
        if code == N.SK_OVERSIZED:
            raise IllegalWorkgroupSize(msg)
        raise N.NativeError(code, where, N.last_error())

    # -- argument checks (the C side copies / reads W*H*sizeof(T) per buffer)
    _TORCH_NAMES = {N.SK_INT32: "int32", N.SK_FLOAT32: "float32", N.SK_FLOAT64: "float64"}

    def _check_device(self, *tensors) -> None:
        want = self._TORCH_NAMES[self._desc.dtype]
        shape = None
        for t in tensors:
            if not getattr(t, "is_cuda", False):
                raise ValueError("stencil buffers must be CUDA tensors")
            if str(t.dtype).split(".")[-1] != want:
                raise ValueError(f"buffer dtype {t.dtype} does not match the stencil's {want}")
            if t.dim() != 2 or t.stride(1) != 1:
                raise ValueError("stencil buffers must be 2-D with unit column stride")
            if shape is not None and t.shape[1] != shape[1]:
                raise ValueError(f"buffer widths differ: {tuple(t.shape)} vs {shape}")
            shape = tuple(t.shape)

    def _check_host(self, h_in, h_out) -> None:
        import numpy as np

        want = np.dtype(self._TORCH_NAMES[self._desc.dtype])
        for a in (h_in, h_out):
            if hasattr(a, "data_ptr"):
                if a.is_cuda or not a.is_contiguous():
                    raise ValueError("host buffers must be contiguous CPU tensors")
                dt = np.dtype(str(a.dtype).split(".")[-1])
            else:
                if not a.flags["C_CONTIGUOUS"]:
                    raise ValueError("host buffers must be C-contiguous")
                dt = np.dtype(a.dtype)
            if dt != want:
                raise ValueError(f"host buffer dtype {dt} does not match the stencil's {want}")
            if len(a.shape) != 2:
                raise ValueError("host buffers must be 2-D")
        if tuple(h_in.shape) != tuple(h_out.shape):
            raise ValueError(f"host buffer shapes differ: {tuple(h_in.shape)} vs {tuple(h_out.shape)}")

    def launch_ptr(self, d_in: int, d_out: int, width: int, height: int, pitch_in: int,
                   pitch_out: int, wc: int, wr: int, rows_above: int = 0, rows_below: int = 0,
                   stream: int = 0) -> None:
        rc = N.lib().sk_stencil_launch(ctypes.byref(self._desc), d_in, d_out, width, height,
                                       pitch_in, pitch_out, rows_above, rows_below, wc, wr,
                                       stream or None)
        if rc:
            self._raise(rc, "sk_stencil_launch", wc, wr)

    def __call__(self, inp, out, wc: int, wr: int, rows_above: int = 0, rows_below: int = 0,
                 height: int | None = None, stream=None) -> None:
        """One pass from torch tensor ``inp`` to ``out`` (row 0 of both at [0])."""
        import torch

        self._check_device(inp, out)
        h = out.shape[0] if height is None else height
        # rows_above halo rows sit before inp's first row (not checkable here)
        if h < 0 or h > out.shape[0] or rows_above < 0 or rows_below < 0 or \
                inp.shape[0] < h + rows_below:
            raise ValueError("height / halo rows exceed the buffers")
        s = (stream or torch.cuda.current_stream(inp.device)).cuda_stream
        self.launch_ptr(inp.data_ptr(), out.data_ptr(), out.shape[1], h, inp.stride(0),
                        out.stride(0), wc, wr, rows_above, rows_below, s)

    def iterate(self, a, b, iterations: int, wc: int, wr: int, stream=None):
        """``iterations`` ping-pong passes; returns the tensor holding the result."""
        import torch

        self._check_device(a, b)
        if tuple(a.shape) != tuple(b.shape) or a.stride(0) != b.stride(0):
            raise ValueError("iterate needs two buffers of the same shape and pitch")
        s = (stream or torch.cuda.current_stream(a.device)).cuda_stream
        in_b = ctypes.c_int32(0)
        rc = N.lib().sk_stencil_iterate(ctypes.byref(self._desc), a.data_ptr(), b.data_ptr(),
                                        a.shape[1], a.shape[0], a.stride(0), iterations, wc, wr,
                                        s or None, ctypes.byref(in_b))
        if rc:
            self._raise(rc, "sk_stencil_iterate", wc, wr)
        return b if in_b.value else a

    def probe(self, width: int, height: int, wc: int, wr: int) -> dict:
        """Zero-work legality probe: {'status', 'kernel_max', 'tile_bytes', 'load_path'}."""
        km, tb, lp = ctypes.c_int32(0), ctypes.c_int64(0), ctypes.c_int32(0)
        rc = N.lib().sk_stencil_probe(ctypes.byref(self._desc), width, height, wc, wr,
                                      ctypes.byref(km), ctypes.byref(tb), ctypes.byref(lp))
        if rc not in (N.SK_OK, N.SK_OVERSIZED, N.SK_REFUSED):
            raise N.NativeError(rc, "sk_stencil_probe", N.last_error())
        return {"status": N.STATUS_NAMES[rc], "kernel_max": km.value, "tile_bytes": tb.value,
                "load_path": {N.SK_LOAD_TMA: "tma", N.SK_LOAD_BITPLANE: "bitplane",
                              N.SK_LOAD_STRIPS: "strips", N.SK_LOAD_VECTOR: "vector"}.get(
                    lp.value, "explicit")}

    def kernel_max(self) -> int:
        km = ctypes.c_int32(0)
        N.check(N.lib().sk_kernel_max_wgsize(ctypes.byref(self._desc), ctypes.byref(km)),
                "sk_kernel_max_wgsize")
        return km.value

    def time(self, inp, out, wc: int, wr: int, samples: int = 30, warmup: int = 3,
             flush_l2: bool = True) -> list[float]:
        """``samples`` cudaEvent-timed passes (ms), after ``warmup`` untimed ones."""
        self._check_device(inp, out)
        if inp.shape[0] < out.shape[0]:
            raise ValueError("input has fewer rows than the output")
        ms = (ctypes.c_double * max(samples, 1))()
        rc = N.lib().sk_stencil_time(ctypes.byref(self._desc), inp.data_ptr(), out.data_ptr(),
                                     out.shape[1], out.shape[0], inp.stride(0), wc, wr, warmup,
                                     samples, int(flush_l2), ms)
        if rc:
            self._raise(rc, "sk_stencil_time", wc, wr)
        return list(ms[:samples])

    def run_host(self, h_in, h_out, iterations: int, wc: int, wr: int) -> None:
        """End-to-end from host arrays (numpy or pinned torch CPU tensors)."""
        self._check_host(h_in, h_out)
        pin = _host_ptr(h_in)
        pout = _host_ptr(h_out)
        height, width = h_in.shape
        rc = N.lib().sk_stencil_run_host(ctypes.byref(self._desc), pin, pout, width, height,
                                         iterations, wc, wr)
        if rc:
            self._raise(rc, "sk_stencil_run_host", wc, wr)


    def submit_host(self, h_in, h_out, iterations: int, wc: int, wr: int) -> int:
        """Streamed end-to-end job (pinned host buffers): returns a ticket
        immediately; at most three jobs are in flight per thread."""
        self._check_host(h_in, h_out)
        t = ctypes.c_int64(-1)
        height, width = h_in.shape
        rc = N.lib().sk_stencil_submit_host(ctypes.byref(self._desc), _host_ptr(h_in),
                                            _host_ptr(h_out), width, height, iterations, wc, wr,
                                            ctypes.byref(t))
        if rc:
            self._raise(rc, "sk_stencil_submit_host", wc, wr)
        return t.value

    @staticmethod
    def wait_host(ticket: int) -> None:
        N.check(N.lib().sk_stencil_wait_host(ticket), "sk_stencil_wait_host")


def _host_ptr(a) -> int:
    if hasattr(a, "data_ptr"):
        return a.data_ptr()
    return a.ctypes.data


def device_features(device: int = 0) -> dict:
    """DeviceDescriptor fields from cudaDeviceProp (north-star subsystem 3)."""
    p = N.sk_device_props()
    N.check(N.lib().sk_device_features(device, ctypes.byref(p)), "sk_device_features")
    out = {f: getattr(p, f) for f, _ in N.sk_device_props._fields_}
    out["name"] = p.name.decode()
    return out


def copy_time(src, dst, samples: int = 30, warmup: int = 3, flush_l2: bool = True,
              kind: str = "kernel") -> list[float]:
    """The streaming ceiling at a given size: ``samples`` timed copies (ms) of
    ``src`` into ``dst`` (device tensors of equal size) under
    ``Stencil.time``'s harness - same stream, events and L2 scrub.  ``kind``
    "kernel" is a 16-B vector copy kernel, "memcpy" cudaMemcpyAsync."""
    if src.device.type != "cuda" or dst.device != src.device:
        raise ValueError("copy_time needs two tensors on the same CUDA device")
    nbytes = src.numel() * src.element_size()
    if dst.numel() * dst.element_size() != nbytes or not (src.is_contiguous() and dst.is_contiguous()):
        raise ValueError("copy_time needs contiguous tensors of equal size")
    ms = (ctypes.c_double * max(samples, 1))()
    N.check(N.lib().sk_copy_time(src.data_ptr(), dst.data_ptr(), nbytes, {"memcpy": 0, "kernel": 1}[kind],
                                 warmup, samples, int(flush_l2), ms), "sk_copy_time")
    return list(ms[:samples])


def fill_host(arr, kind: int, seed: int) -> None:
    """Deterministic reference-Rng input (mt19937_64, rng.hpp:34-72) into a host array."""
    import numpy as np

    code = {np.dtype("int32"): N.SK_INT32, np.dtype("float32"): N.SK_FLOAT32,
            np.dtype("float64"): N.SK_FLOAT64}[np.dtype(arr.dtype)]
    assert arr.flags["C_CONTIGUOUS"]
    N.check(N.lib().sk_fill_host(code, kind, seed, arr.ctypes.data, arr.size), "sk_fill_host")
