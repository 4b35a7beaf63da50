"""GPU parity of the register-strip temporally blocked cross stencils
(csrc/stencil/cross_strips.cuh, SK_LOAD_STRIPS: five_point and heat with unit
borders) against the CPU oracle: TB generations per launch must equal TB
single passes bit for bit, for every element type, border mode and pad
value, ragged widths (not a multiple of 4, narrower than one lane group),
unaligned pitches (scalar loads), block shapes including partial warps, TB
across the 4-column lane boundary, and row-shard halos."""
from __future__ import annotations

import numpy as np
import pytest

import oracle_lib as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_1511_02490_b200 import IllegalWorkgroupSize, RefusedParameter, Stencil  # noqa: E402

TDT = {"int32": torch.int32, "float32": torch.float32, "float64": torch.float64}


def grid(dtype, shape, seed):
    rng = np.random.default_rng(seed)
    if dtype == "int32":
        return rng.integers(-1000, 1000, size=shape).astype(np.int32)
    return (2 * rng.random(shape) - 1).astype(dtype)


def strips(op, dtype, tb, k=0, border="nearest", pad=0.0):
    return Stencil(op=op, dtype=dtype, border=border, pad_value=pad, load_path="strips",
                   fused_iterations=tb, cells_per_thread=k)


def tile_fits(tb, wc, wr, k, dtype="float32"):
    """ceil(wc*wr/32) warps x R rows (R = k, or 8 / 4 for float64) must hold
    2*TB halo rows plus one output row."""
    return ((wc * wr + 31) // 32) * (k or (4 if dtype == "float64" else 8)) > 2 * tb


def run(st, x, iters, wc, wr, pitch_pad=0):
    """Iterate on the GPU; `pitch_pad` extra columns make the row pitch
    unaligned (the scalar-load path)."""
    h, w = x.shape
    buf = np.zeros((h, w + pitch_pad), dtype=x.dtype)
    buf[:, :w] = x
    a = torch.from_numpy(buf).cuda()[:, :w]
    b = torch.empty_like(torch.from_numpy(buf)).cuda()[:, :w]
    res = st.iterate(a, b, iters, wc, wr)
    torch.cuda.synchronize()
    return res.cpu().numpy()


def oracle(st, x, iters):
    return O.iterate(O.desc_from_stencil(st), x, iters)


@pytest.mark.parametrize("k", [0, 4, 8])
@pytest.mark.parametrize("dtype", ["int32", "float32", "float64"])
@pytest.mark.parametrize("op", ["heat", "five_point"])
@pytest.mark.parametrize("border,pad", [("pad", 0.0), ("pad", 1.5), ("nearest", 0.0)])
@pytest.mark.parametrize("shape", [(37, 20), (64, 64), (101, 301), (130, 1000)])
def test_strips_vs_oracle(op, dtype, border, pad, shape, k):
    x = grid(dtype, shape, seed=shape[0] * 7 + shape[1])
    for iters, tb, wc, wr in [(1, 1, 8, 8), (5, 2, 2, 16), (9, 4, 32, 8), (11, 5, 32, 4),
                              (12, 12, 32, 16), (7, 3, 3, 5)]:
        st = strips(op, dtype, tb, k, border, pad)
        if st.probe(shape[1], shape[0], wc, wr)["status"] != "OK":
            assert not tile_fits(min(tb, iters), wc, wr, k, dtype) or wc * wr > st.kernel_max()
            continue
        got = run(st, x, iters, wc, wr)
        want = oracle(st, x, iters)
        assert got.tobytes() == want.tobytes(), f"{op} {dtype} {border}/{pad} {shape} it={iters} tb={tb} {wc}x{wr}"


@pytest.mark.parametrize("dtype", ["int32", "float32"])
@pytest.mark.parametrize("tb", [1, 3, 4, 5, 8, 9, 16, 32])
def test_strips_generation_counts(dtype, tb):
    x = grid(dtype, (300, 520), seed=tb)
    for border in ("pad", "nearest"):
        st = strips("heat", dtype, tb, 16, border)
        if not tile_fits(min(tb, 50), 32, 12, 16):
            assert st.probe(520, 300, 32, 12)["status"] == "REFUSED"
            continue
        got = run(st, x, 50, 32, 12)
        assert got.tobytes() == oracle(st, x, 50).tobytes(), f"tb={tb} {border}"


@pytest.mark.parametrize("pitch_pad", [1, 2, 3])
def test_strips_unaligned_pitch(pitch_pad):
    x = grid("float32", (90, 203), seed=pitch_pad)
    st = strips("heat", "float32", 6, 8, "nearest")
    got = run(st, x, 13, 32, 8, pitch_pad=pitch_pad)
    assert got.tobytes() == oracle(st, x, 13).tobytes()


@pytest.mark.parametrize("wc,wr", [(1, 1), (2, 2), (4, 64), (32, 12), (64, 6), (384, 1),
                                   (7, 9), (100, 5), (32, 32)])
@pytest.mark.parametrize("k", [0, 4, 8, 16])
def test_strips_block_shapes(wc, wr, k):
    x = grid("float32", (257, 700), seed=wc * 31 + wr)
    st = strips("heat", "float32", 6, k, "nearest")
    status = st.probe(700, 257, wc, wr)["status"]
    if status != "OK":
        # a refusal must be the planned one: a tile too short for the halo
        # rows, or more threads than the kernel's register budget allows
        assert (status == "REFUSED" and not tile_fits(6, wc, wr, k)) or \
               (status == "OVERSIZED" and wc * wr > st.kernel_max())
        a = torch.zeros((64, 64), dtype=torch.float32, device="cuda")
        with pytest.raises((RefusedParameter, IllegalWorkgroupSize)):
            st.iterate(a, torch.empty_like(a), 6, wc, wr)
        return
    got = run(st, x, 20, wc, wr)
    assert got.tobytes() == oracle(st, x, 20).tobytes(), f"{wc}x{wr} K={k}"


def test_strips_config3_matches_one_pass():
    """BASELINE config 3 shape (16384^2 f32 heat, nearest): 24 generations on
    the strip path equal 24 single passes of the per-cell executor (a
    size-independent property; the oracle is checked at reduced size)."""
    from paper_1511_02490_b200 import fill_host

    host = np.empty((16384, 16384), dtype=np.float32)
    fill_host(host, 1, 3)
    a = torch.from_numpy(host).cuda()
    one = Stencil(op="heat", dtype="float32", border="nearest")
    want = one.iterate(a.clone(), torch.empty_like(a), 24, 64, 8).clone()
    st = strips("heat", "float32", 8, 16, "nearest")
    b = torch.empty_like(a)
    got = st.iterate(a, b, 24, 32, 12)
    torch.cuda.synchronize()
    assert torch.equal(got, want)


def test_strips_halo_rows_match_full_grid():
    """A row shard with TB-deep halos advances TB generations exactly like the
    same rows of the undivided grid (the temporally blocked multi-GPU exchange
    relies on this)."""
    x = grid("float32", (200, 333), seed=3)
    tb = 6
    for border, k in (("pad", 0), ("nearest", 0), ("pad", 8), ("nearest", 4)):
        st = strips("heat", "float32", tb, k, border)
        want = oracle(st, x, tb)
        for r0, r1 in [(0, 70), (70, 150), (150, 200), (3, 5)]:
            above, below = min(tb, r0), min(tb, 200 - r1)
            win = torch.from_numpy(np.ascontiguousarray(x[r0 - above:r1 + below])).cuda()
            out = torch.zeros((r1 - r0, 333), dtype=torch.float32, device="cuda")
            st(win[above:], out, 32, 8, rows_above=above, rows_below=below, height=r1 - r0)
            torch.cuda.synchronize()
            assert out.cpu().numpy().tobytes() == want[r0:r1].tobytes(), f"{border} rows {r0}:{r1}"


def test_strips_auto_and_legality():
    auto = Stencil(op="heat", dtype="float32", border="nearest", fused_iterations=8)
    assert auto.probe(4096, 4096, 32, 12)["load_path"] == "strips"
    assert Stencil(op="heat", dtype="float32", fused_iterations=4).probe(
        4096, 4096, 32, 8)["load_path"] == "tma"  # TB <= 4: the per-cell fused kernel
    st = strips("heat", "float32", 8)
    km = st.kernel_max()
    assert km < 1024  # register-bound per-kernel maximum (R = 8 rows per lane: 384)
    assert st.probe(4096, 4096, 32, 32)["status"] == "OVERSIZED"
    # 1 warp x 4 rows cannot hold 2 x 8 halo rows
    assert strips("heat", "float32", 8, 4).probe(4096, 4096, 32, 1)["status"] == "REFUSED"
    with pytest.raises(Exception):  # only unit-border cross ops
        Stencil(op="gol", dtype="int32", load_path="strips").probe(64, 64, 32, 8)
    with pytest.raises(Exception):
        Stencil(op="heat", dtype="float32", north=2, load_path="strips").probe(64, 64, 32, 8)
    with pytest.raises(Exception):
        strips("heat", "float32", 33).probe(64, 64, 32, 8)


@pytest.mark.parametrize("op", ["heat", "five_point"])
def test_strips_subnormals_and_signed_zeros(op):
    """The fp32 pair path (packed FADD2 + scalar products) must round exactly
    like the scalar executor on subnormal inputs, signed zeros and large
    magnitudes as well."""
    rng = np.random.default_rng(9)
    x = (rng.standard_normal((70, 260)) * 1e-39).astype(np.float32)  # subnormal range
    x[::7] = -0.0
    x[3::11] = rng.standard_normal(x[3::11].shape).astype(np.float32) * 1e30
    for border, pad in (("nearest", 0.0), ("pad", -0.0)):
        st = strips(op, "float32", 5, 8, border, pad)
        got = run(st, x, 11, 32, 8)
        assert got.tobytes() == oracle(st, x, 11).tobytes(), border
