"""Pins the CPU stencil oracle (oracle/stencil_oracle.c) before it is trusted.

The reference has no stencil implementation or golden grids,
so the oracle is pinned by (1) analytic known answers and (2) the independent
numpy restatement committed in tests/golden/stencil_golden.npz
(tests/golden/make_golden.py).  All comparisons are bit-exact.
"""
from __future__ import annotations

from pathlib import Path

import numpy as np
import pytest

import oracle_lib as O

GOLDEN = Path(__file__).resolve().parent / "golden" / "stencil_golden.npz"


def gol(grid, gens, border="pad"):
    d = O.desc_from("gol", "int32", border=border)
    return O.iterate(d, grid.astype(np.int32), gens)


def place(shape, cells, r0=0, c0=0):
    g = np.zeros(shape, np.int32)
    for r, c in cells:
        g[r0 + r, c0 + c] = 1
    return g


def test_gol_block_is_still_life():
    g = place((8, 8), [(0, 0), (0, 1), (1, 0), (1, 1)], 3, 3)
    for gens in (1, 2, 7):
        np.testing.assert_array_equal(gol(g, gens), g)


def test_gol_blinker_has_period_two():
    g = place((9, 9), [(0, 0), (0, 1), (0, 2)], 4, 3)
    g1 = gol(g, 1)
    np.testing.assert_array_equal(g1, place((9, 9), [(0, 0), (1, 0), (2, 0)], 3, 4))
    np.testing.assert_array_equal(gol(g, 2), g)


def test_gol_glider_translates_diagonally():
    glider = [(0, 1), (1, 2), (2, 0), (2, 1), (2, 2)]
    g = place((20, 24), glider, 2, 2)
    for k in (1, 2, 3):
        np.testing.assert_array_equal(gol(g, 4 * k), place((20, 24), glider, 2 + k, 2 + k))


def test_gol_pad_zero_is_dead_boundary():
    # A blinker touching the north edge: with dead (pad 0) cells outside the
    # matrix it still oscillates as in the infinite plane, clipped.
    g = place((6, 6), [(0, 1), (0, 2), (0, 3)])
    g1 = gol(g, 1)
    np.testing.assert_array_equal(g1, place((6, 6), [(0, 2), (1, 2)]))


def test_heat_constant_field_is_fixed_point_nearest():
    for dt in ("float32", "float64", "int32"):
        g = np.full((17, 13), 3, dtype=dt)
        d = O.desc_from("heat", dt, border="nearest")
        np.testing.assert_array_equal(O.iterate(d, g, 5), g)


def test_five_point_delta_response_pad0():
    g = np.zeros((9, 9), np.float32)
    g[4, 4] = 1.0
    out = O.stencil(O.desc_from("five_point", "float32"), g)
    want = np.zeros_like(g)
    for r, c in ((4, 4), (3, 4), (5, 4), (4, 3), (4, 5)):
        want[r, c] = np.float32(1.0) * np.float32(0.2)
    np.testing.assert_array_equal(out, want)


def test_asymmetric_boxmean_nearest_on_ramps():
    # N=5, S=1, E=3, W=0 (BASELINE config 4): column ramp checks the east clamp,
    # row ramp the north/south clamps.
    H, W = 12, 10
    d = O.desc_from("boxmean", "float64", 5, 1, 3, 0, border="nearest")
    cols = np.tile(np.arange(W, dtype=np.float64), (H, 1))
    out = O.stencil(d, cols)
    for c in range(W):
        taps = [min(c + k, W - 1) for k in range(4)]
        np.testing.assert_allclose(out[:, c], np.mean(taps), rtol=0, atol=1e-12)
    rows = np.tile(np.arange(H, dtype=np.float64)[:, None], (1, W))
    out = O.stencil(d, rows)
    for r in range(H):
        taps = [min(max(r + k, 0), H - 1) for k in range(-5, 2)]
        np.testing.assert_allclose(out[r, :], np.mean(taps), rtol=0, atol=1e-12)


def test_pad_value_is_used_outside():
    g = np.zeros((4, 5), np.float32)
    d = O.desc_from("boxmean", "float32", 1, 1, 1, 1, border="pad", pad=9.0)
    out = O.stencil(d, g)
    # corner cell sees 5 pad cells of 9 out of 9 taps
    assert out[0, 0] == np.float32(45.0) / np.float32(9.0)
    assert out[1, 1] == 0.0


def test_halo_rows_are_real_data():
    # A shard with halo rows above/below must equal the matching rows of the
    # full-grid pass (the row-block decomposition invariant).
    rng = np.random.default_rng(3)
    full = rng.random((40, 33)).astype(np.float32)
    d = O.desc_from("boxmean", "float32", 3, 2, 1, 2, border="nearest")
    want = O.stencil(d, full)
    r0, r1 = 11, 27
    shard = full[r0 - 3:r1 + 2]
    got = O.stencil(d, shard, rows_above=3, rows_below=2)
    np.testing.assert_array_equal(got, want[r0:r1])
    # first shard: no rows above -> nearest clamp to global row 0
    got0 = O.stencil(d, full[0:r1 + 2], rows_above=0, rows_below=2)
    np.testing.assert_array_equal(got0, want[0:r1])


def golden_cases():
    z = np.load(GOLDEN)
    names = sorted({k.split("__")[0] for k in z.files})
    return [(n, z) for n in names]


@pytest.mark.parametrize("name", [n for n, _ in golden_cases()])
def test_oracle_matches_numpy_golden(name):
    z = np.load(GOLDEN)
    x, y = z[f"{name}__in"], z[f"{name}__out"]
    n, s, e, w, nearest, cx, ins = (int(v) for v in z[f"{name}__meta"])
    op = str(z[f"{name}__op"])
    d = O.desc_from(op, x.dtype, n, s, e, w, "nearest" if nearest else "pad",
                    float(z[f"{name}__pad"][0]), cx, ins)
    for threads in (1, 4):
        out = O.stencil(d, x, threads=threads)
        assert out.dtype == y.dtype
        assert out.tobytes() == y.tobytes(), f"{name}: oracle differs from numpy golden"


# ----------------------------------------------------------- input + baseline
def test_oracle_fill_matches_mt19937_64():
    # std::mt19937_64 default seed 5489: 10000th output is 9981545732273789042
    # (C++11 [rand.predef]); first output 14514284786278117030.
    a = O.fill((4,), "float64", 1, 5489)
    assert a[0] == (14514284786278117030 >> 11) * 2.0 ** -53
    b = O.fill((10000,), "float64", 1, 5489)
    assert b[-1] == (9981545732273789042 >> 11) * 2.0 ** -53
    g = O.fill((64, 64), "int32", 2, 2)
    assert set(np.unique(g)) <= {0, 1} and 1500 < g.sum() < 2600
    f = O.fill((1000,), "float32", 0, 1)
    assert f.min() >= -1.0 and f.max() <= 1.0


@pytest.mark.parametrize("op,dtype,borders,border,pad", [
    ("gol", "int32", (1, 1, 1, 1), "pad", 0.0),
    ("gol", "int32", (1, 1, 1, 1), "nearest", 0.0),
    ("heat", "float32", (1, 1, 1, 1), "nearest", 0.0),
    ("heat", "float32", (1, 1, 1, 1), "pad", 0.5),
    ("five_point", "float32", (1, 1, 1, 1), "pad", 0.0),
    ("five_point", "float32", (1, 1, 1, 1), "pad", 1.0),
    ("boxmean", "float32", (5, 1, 3, 0), "nearest", 0.0),
    ("boxmean", "float32", (2, 3, 0, 4), "pad", -1.5),
    ("sobel", "float32", (1, 1, 1, 1), "nearest", 0.0),   # no fast path: per-cell
    ("heat", "float64", (1, 1, 1, 1), "nearest", 0.0),
])
@pytest.mark.parametrize("shape", [(1, 1), (2, 9), (7, 3), (37, 129), (130, 67)])
def test_baseline_is_bit_identical_to_oracle(op, dtype, borders, border, pad, shape):
    n, s, e, w = borders
    d = O.desc_from(op, dtype, n, s, e, w, border, pad)
    kind = 2 if op == "gol" else 0
    g = O.fill(shape, dtype, kind, 11 + shape[0])
    want = O.iterate(d, g, 3, threads=3)
    got = O.baseline_iterate(d, g, 3, threads=3)
    assert got.tobytes() == want.tobytes()


def test_baseline_special_values_bit_identical():
    d = O.desc_from("heat", "float32", border="nearest")
    g = O.fill((33, 70), "float32", 0, 4)
    g[3, 5], g[10, 10], g[20, 30] = np.inf, -np.nan, -0.0
    g[5, 6] = 1e-40  # subnormal
    assert O.baseline_stencil(d, g).tobytes() == O.stencil(d, g).tobytes()
