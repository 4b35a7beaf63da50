"""Test-side loader for the CPU oracle (oracle/stencil_oracle.c).

Test infrastructure only: the oracle is the checker, never the thing measured
or shipped.  Builds oracle/_build/liboracle_stencil.so with make if missing.
"""
from __future__ import annotations

import ctypes
import subprocess
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
ORACLE_DIR = ROOT / "oracle"
LIB = ORACLE_DIR / "_build" / "liboracle_stencil.so"

_lib = None

OPS = {"five_point": 0, "heat": 1, "gol": 2, "boxmean": 3, "gaussian": 4, "sobel": 5, "nms": 6,
       "threshold": 7, "synthetic": 8}
DT = {np.dtype("int32"): 0, np.dtype("float32"): 1, np.dtype("float64"): 2}


class oracle_desc(ctypes.Structure):
    _fields_ = [("op", ctypes.c_int32), ("dtype", ctypes.c_int32), ("north", ctypes.c_int32),
                ("south", ctypes.c_int32), ("east", ctypes.c_int32), ("west", ctypes.c_int32),
                ("border_mode", ctypes.c_int32), ("pad_value", ctypes.c_double),
                ("complexity", ctypes.c_int32), ("instructions", ctypes.c_int32),
                ("load_path", ctypes.c_int32), ("cells_per_thread", ctypes.c_int32),
                ("fused_iterations", ctypes.c_int32)]


def lib():
    global _lib
    if _lib is None:
        if not LIB.exists():
            subprocess.run(["make", "-s", "-C", str(ORACLE_DIR)], check=True)
        _lib = ctypes.CDLL(str(LIB))
        _lib.oracle_stencil.restype = ctypes.c_int
        _lib.oracle_stencil.argtypes = [ctypes.POINTER(oracle_desc), ctypes.c_void_p,
                                        ctypes.c_void_p] + [ctypes.c_int64] * 6 + [ctypes.c_int32]
        _lib.oracle_iterate.restype = ctypes.c_int
        _lib.oracle_iterate.argtypes = [ctypes.POINTER(oracle_desc), ctypes.c_void_p,
                                        ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                                        ctypes.c_int32, ctypes.c_int32]
        _lib.oracle_fill.restype = ctypes.c_int
        _lib.oracle_fill.argtypes = [ctypes.c_int32, ctypes.c_int32, ctypes.c_uint64,
                                     ctypes.c_void_p, ctypes.c_int64]
        _lib.oracle_baseline_stencil.restype = ctypes.c_int
        _lib.oracle_baseline_stencil.argtypes = [ctypes.POINTER(oracle_desc), ctypes.c_void_p,
                                                 ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                                                 ctypes.c_int32]
        _lib.oracle_baseline_iterate.restype = ctypes.c_int
        _lib.oracle_baseline_iterate.argtypes = _lib.oracle_iterate.argtypes
    return _lib


def fill(shape, dtype, kind: int, seed: int) -> np.ndarray:
    """The bench/test input stream (reference Rng, mt19937_64) without the
    product library: kind 0 -> 2u-1, 1 -> u, 2 -> u<0.5, 3 -> floor(256u)."""
    a = np.empty(shape, dtype=dtype)
    rc = lib().oracle_fill(DT[np.dtype(dtype)], kind, seed, a.ctypes.data, a.size)
    assert rc == 0, "oracle_fill rejected arguments"
    return a


def baseline_stencil(desc: oracle_desc, grid: np.ndarray, threads: int = 8) -> np.ndarray:
    """One pass of the vectorised CPU baseline (bit-identical to stencil())."""
    grid = np.ascontiguousarray(grid)
    out = np.empty_like(grid)
    rc = lib().oracle_baseline_stencil(ctypes.byref(desc), grid.ctypes.data, out.ctypes.data,
                                       grid.shape[1], grid.shape[0], threads)
    assert rc == 0
    return out


def baseline_iterate(desc: oracle_desc, grid: np.ndarray, iterations: int,
                     threads: int = 8) -> np.ndarray:
    a = np.ascontiguousarray(grid).copy()
    b = np.empty_like(a)
    rc = lib().oracle_baseline_iterate(ctypes.byref(desc), a.ctypes.data, b.ctypes.data,
                                       a.shape[1], a.shape[0], iterations, threads)
    assert rc == 0
    return b if iterations % 2 else a


def desc_from(op, dtype, n=1, s=1, e=1, w=1, border="pad", pad=0.0, complexity=0,
              instructions=100):
    return oracle_desc(op=OPS[op], dtype=DT[np.dtype(dtype)], north=n, south=s, east=e, west=w,
                       border_mode=1 if border == "nearest" else 0, pad_value=float(pad),
                       complexity=complexity, instructions=instructions, load_path=0)


def desc_from_stencil(st) -> oracle_desc:
    d = st.desc
    return oracle_desc(op=d.op, dtype=d.dtype, north=d.north, south=d.south, east=d.east,
                       west=d.west, border_mode=d.border_mode, pad_value=d.pad_value,
                       complexity=d.complexity, instructions=d.instructions, load_path=0)


def stencil(desc: oracle_desc, grid: np.ndarray, rows_above: int = 0, rows_below: int = 0,
            threads: int = 8) -> np.ndarray:
    """One pass.  `grid` holds rows_above + H + rows_below rows; returns H x W."""
    grid = np.ascontiguousarray(grid)
    h = grid.shape[0] - rows_above - rows_below
    w = grid.shape[1]
    out = np.empty((h, w), dtype=grid.dtype)
    base = grid.ctypes.data + rows_above * grid.strides[0]
    rc = lib().oracle_stencil(ctypes.byref(desc), base, out.ctypes.data, w, h, w, w,
                              rows_above, rows_below, threads)
    assert rc == 0, "oracle rejected arguments"
    return out


def iterate(desc: oracle_desc, grid: np.ndarray, iterations: int, threads: int = 8) -> np.ndarray:
    a = np.ascontiguousarray(grid).copy()
    b = np.empty_like(a)
    rc = lib().oracle_iterate(ctypes.byref(desc), a.ctypes.data, b.ctypes.data, a.shape[1],
                              a.shape[0], iterations, threads)
    assert rc == 0
    return b if iterations % 2 else a
