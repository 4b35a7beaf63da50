"""Generate tests/golden/stencil_golden.npz — an independent numpy restatement
of the stencil semantics and of the customising functions
of DESIGN.md §3, written without reference to oracle/stencil_oracle.c or the
CUDA kernels.  The CPU oracle is checked against these fixtures
(tests/test_oracle_kat.py) and the GPU executor against both
(tests/test_stencil_parity.py).

Border handling here is np.pad: mode "edge" is the nearest-cell rule,
"constant" the pad-value rule.  North = smaller row index, east = larger
column index.

Run:  python tests/golden/make_golden.py
"""
from __future__ import annotations

from pathlib import Path

import numpy as np

OUT = Path(__file__).resolve().parent / "stencil_golden.npz"


def padded(grid, n, s, e, w, border, pad):
    if border == "nearest":
        return np.pad(grid, ((n, s), (w, e)), mode="edge")
    return np.pad(grid, ((n, s), (w, e)), mode="constant",
                  constant_values=grid.dtype.type(pad))


def trunc_div(a, b):
    """C integer division (truncation toward zero) on int64 arrays."""
    q = np.abs(a) // b
    return np.where(a < 0, -q, q)


def run(op, grid, n, s, e, w, border="pad", pad=0.0, complexity=0, instructions=100):
    H, W = grid.shape
    P = padded(grid, n, s, e, w, border, pad)
    dt = grid.dtype
    isint = dt == np.int32
    f = dt.type

    def v(dr, dc):
        x = P[n + dr:n + dr + H, w + dc:w + dc + W]
        return x.astype(np.int64) if isint else x

    if op == "five_point":
        if isint:
            return trunc_div(v(-1, 0) + v(1, 0) + v(0, 1) + v(0, -1) + v(0, 0), 5).astype(dt)
        t = v(-1, 0) + v(1, 0)
        t = t + v(0, 1)
        t = t + v(0, -1)
        t = t + v(0, 0)
        return t * f(0.2)
    if op == "heat":
        u = v(0, 0)
        if isint:
            lap = v(-1, 0) + v(1, 0) + v(0, 1) + v(0, -1) - 4 * u
            return (u + trunc_div(lap, 5)).astype(dt)
        lap = v(-1, 0) + v(1, 0)
        lap = lap + v(0, 1)
        lap = lap + v(0, -1)
        lap = lap - f(4) * u
        return u + f(0.2) * lap
    if op == "gol":
        cnt = sum((v(dr, dc) != 0).astype(np.int32) for dr in (-1, 0, 1) for dc in (-1, 0, 1)
                  if dr or dc)
        alive = v(0, 0) != 0
        return np.where((cnt == 3) | (alive & (cnt == 2)), 1, 0).astype(dt)
    if op == "boxmean":  # sum of row sums (west->east), rows north->south
        acc = None
        for dr in range(-n, s + 1):
            row = v(dr, -w)
            for dc in range(-w + 1, e + 1):
                row = row + v(dr, dc)
            acc = row if acc is None else acc + row
        cnt = (n + s + 1) * (e + w + 1)
        return trunc_div(acc, cnt).astype(dt) if isint else acc / f(cnt)
    if op == "gaussian":
        g = n
        from math import comb
        # separable: row pass west->east, then the rows north->south
        b = [comb(2 * g, g + j) for j in range(-g, g + 1)]
        bw = [np.int64(c) if isint else f(np.ldexp(float(c), -2 * g)) for c in b]
        acc = None
        for i in range(-g, g + 1):
            row = bw[0] * v(i, -g)
            for j in range(-g + 1, g + 1):
                row = row + bw[j + g] * v(i, j)
            t = bw[i + g] * row
            acc = t if acc is None else acc + t
        return (acc >> (4 * g)).astype(dt) if isint else acc
    if op == "sobel":
        if isint:
            gx = (v(-1, 1) + 2 * v(0, 1) + v(1, 1)) - (v(-1, -1) + 2 * v(0, -1) + v(1, -1))
            gy = (v(1, -1) + 2 * v(1, 0) + v(1, 1)) - (v(-1, -1) + 2 * v(-1, 0) + v(-1, 1))
            return (np.abs(gx) + np.abs(gy)).astype(dt)
        ex = v(-1, 1) + f(2) * v(0, 1)
        ex = ex + v(1, 1)
        wx = v(-1, -1) + f(2) * v(0, -1)
        wx = wx + v(1, -1)
        gx = ex - wx
        sy = v(1, -1) + f(2) * v(1, 0)
        sy = sy + v(1, 1)
        ny = v(-1, -1) + f(2) * v(-1, 0)
        ny = ny + v(-1, 1)
        gy = sy - ny
        m2 = gx * gx
        m2 = m2 + gy * gy
        return np.sqrt(m2)
    if op == "nms":
        m = v(-1, -1)
        for dr, dc in ((-1, 0), (-1, 1), (0, -1), (0, 1), (1, -1), (1, 0), (1, 1)):
            m = np.maximum(m, v(dr, dc))
        c = v(0, 0)
        return np.where(c >= m, c, 0).astype(dt)
    if op == "threshold":
        return np.where(v(0, 0) > (0 if isint else f(0.5)), 1, 0).astype(dt)
    if op == "synthetic":
        acc = np.zeros((H, W), np.int64 if isint else dt)
        for dr in range(-n, s + 1):
            acc = acc + v(dr, 0)
        for dc in range(-w, 0):
            acc = acc + v(0, dc)
        for dc in range(1, e + 1):
            acc = acc + v(0, dc)
        taps = n + s + 1 + e + w
        iters = (instructions // 4) if complexity else (instructions // 32)
        if isint:
            x = trunc_div(acc, taps).astype(np.int32).astype(np.uint32)
            for _ in range(iters):
                x = x * np.uint32(1664525) + np.uint32(1013904223)
            return x.astype(np.int32)
        x = acc / f(taps)
        for _ in range(iters):
            x = x * f(0.999)
            x = x + f(0.001)
        return x
    raise ValueError(op)


CASES = [
    # (name, op, dtype, n, s, e, w, border, pad, complexity, instructions)
    ("five_point_f32_pad0", "five_point", "float32", 1, 1, 1, 1, "pad", 0.0, 0, 0),
    ("five_point_f32_pad1", "five_point", "float32", 1, 1, 1, 1, "pad", 1.0, 0, 0),
    ("five_point_f64_nearest", "five_point", "float64", 1, 1, 1, 1, "nearest", 0.0, 0, 0),
    ("five_point_i32_pad", "five_point", "int32", 1, 1, 1, 1, "pad", -7.0, 0, 0),
    ("heat_f32_nearest", "heat", "float32", 1, 1, 1, 1, "nearest", 0.0, 0, 0),
    ("heat_f64_pad", "heat", "float64", 1, 1, 1, 1, "pad", 0.25, 0, 0),
    ("heat_i32_nearest", "heat", "int32", 1, 1, 1, 1, "nearest", 0.0, 0, 0),
    ("gol_i32_pad0", "gol", "int32", 1, 1, 1, 1, "pad", 0.0, 0, 0),
    ("gol_i32_nearest", "gol", "int32", 1, 1, 1, 1, "nearest", 0.0, 0, 0),
    ("gol_f32_pad1", "gol", "float32", 1, 1, 1, 1, "pad", 1.0, 0, 0),
    ("boxmean_5130_f32_nearest", "boxmean", "float32", 5, 1, 3, 0, "nearest", 0.0, 0, 0),
    ("boxmean_2304_f64_pad", "boxmean", "float64", 2, 3, 0, 4, "pad", 0.5, 0, 0),
    ("boxmean_5130_i32_pad", "boxmean", "int32", 5, 1, 3, 0, "pad", 3.0, 0, 0),
    ("gaussian_g1_f32_nearest", "gaussian", "float32", 1, 1, 1, 1, "nearest", 0.0, 0, 0),
    ("gaussian_g3_f64_pad", "gaussian", "float64", 3, 3, 3, 3, "pad", 0.0, 0, 0),
    ("gaussian_g5_f32_nearest", "gaussian", "float32", 5, 5, 5, 5, "nearest", 0.0, 0, 0),
    ("gaussian_g5_i32_pad", "gaussian", "int32", 5, 5, 5, 5, "pad", 0.0, 0, 0),
    ("gaussian_g2_i32_nearest", "gaussian", "int32", 2, 2, 2, 2, "nearest", 0.0, 0, 0),
    ("sobel_f32_nearest", "sobel", "float32", 1, 1, 1, 1, "nearest", 0.0, 0, 0),
    ("sobel_i32_pad", "sobel", "int32", 1, 1, 1, 1, "pad", 0.0, 0, 0),
    ("nms_f64_pad", "nms", "float64", 1, 1, 1, 1, "pad", 0.0, 0, 0),
    ("nms_i32_nearest", "nms", "int32", 1, 1, 1, 1, "nearest", 0.0, 0, 0),
    ("threshold_f32_pad", "threshold", "float32", 0, 0, 0, 0, "pad", 0.0, 0, 0),
    ("threshold_i32_pad", "threshold", "int32", 0, 0, 0, 0, "pad", 0.0, 0, 0),
    ("synthetic_a_f32_nearest", "synthetic", "float32", 3, 1, 2, 4, "nearest", 0.0, 0, 100),
    ("synthetic_b_f64_pad", "synthetic", "float64", 2, 5, 1, 3, "pad", 0.0, 1, 600),
    ("synthetic_b_i32_nearest", "synthetic", "int32", 4, 2, 3, 1, "nearest", 0.0, 1, 620),
]


def make_input(dtype, op, rng, shape):
    if dtype == "int32":
        if op == "gol":
            return (rng.random(shape) < 0.4).astype(np.int32)
        return rng.integers(-300, 300, size=shape, dtype=np.int32)
    return (2.0 * rng.random(shape) - 1.0).astype(dtype)


def main():
    rng = np.random.default_rng(1511_02490)
    arrays = {}
    for case in CASES:
        name, op, dtype, n, s, e, w, border, pad, cx, ins = case
        shape = (23, 37)
        x = make_input(dtype, op, rng, shape)
        y = run(op, x, n, s, e, w, border, pad, cx, ins)
        assert y.dtype == np.dtype(dtype), (name, y.dtype)
        arrays[f"{name}__in"] = x
        arrays[f"{name}__out"] = y
        arrays[f"{name}__meta"] = np.array([n, s, e, w, 1 if border == "nearest" else 0, cx, ins],
                                           np.int64)
        arrays[f"{name}__pad"] = np.array([pad], np.float64)
        arrays[f"{name}__op"] = np.array(op)
    np.savez_compressed(OUT, **arrays)
    print(f"wrote {len(CASES)} cases to {OUT}")


if __name__ == "__main__":
    main()
