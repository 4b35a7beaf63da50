"""GPU parity of the bit-sliced, temporally blocked Game of Life kernel
(csrc/stencil/gol_bits.cuh, SK_LOAD_BITPLANE) against the CPU oracle:
TB generations per launch must equal TB single passes bit for bit, for every
element type, border mode, ragged width (not a multiple of 32, narrower than
one word), block shape (including thread counts that are not whole warps),
TB across the 32-generation word boundary and row-shard halos."""
from __future__ import annotations

import numpy as np
import pytest

import oracle_lib as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_1511_02490_b200 import IllegalWorkgroupSize, RefusedParameter, Stencil  # noqa: E402

TDT = {"int32": torch.int32, "float32": torch.float32, "float64": torch.float64}


def grid(dtype, shape, seed, density=0.4):
    """Alive cells are arbitrary non-zero values (the op tests != 0)."""
    rng = np.random.default_rng(seed)
    alive = rng.random(shape) < density
    vals = rng.integers(1, 9, size=shape) * np.where(rng.random(shape) < 0.5, -1, 1)
    return np.where(alive, vals, 0).astype(dtype)


def tile_fits(tb, wc, wr, k):
    """The strip kernel's tile is ceil(wc*wr/32) warps x R rows (R = k or 16)
    and must hold 2*TB halo rows plus at least one output row."""
    return ((wc * wr + 31) // 32) * (k or 16) > 2 * tb


def run_bits(x, iters, tb, wc, wr, border="pad", pad=0.0, k=0, dtype=None):
    dtype = dtype or str(x.dtype)
    st = Stencil(op="gol", dtype=dtype, border=border, pad_value=pad, load_path="bitplane",
                 fused_iterations=tb, cells_per_thread=k)
    status = st.probe(x.shape[1], x.shape[0], wc, wr)["status"]
    if status == "OVERSIZED":  # above the kernel's register-bound maximum
        with pytest.raises(IllegalWorkgroupSize):
            st.iterate(torch.zeros((8, 8), dtype=TDT[dtype], device="cuda"),
                       torch.zeros((8, 8), dtype=TDT[dtype], device="cuda"), iters, wc, wr)
        return st, None
    if not tile_fits(min(tb, iters), wc, wr, k):
        assert status == "REFUSED"
        with pytest.raises(RefusedParameter):
            st.iterate(torch.zeros((8, 8), dtype=TDT[dtype], device="cuda"),
                       torch.zeros((8, 8), dtype=TDT[dtype], device="cuda"), iters, wc, wr)
        return st, None
    a = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    b = torch.empty_like(a)
    res = st.iterate(a, b, iters, wc, wr)
    torch.cuda.synchronize()
    return st, res.cpu().numpy()


def oracle(st, x, iters):
    return O.iterate(O.desc_from_stencil(st), x, iters)


# cells_per_thread on the bit-plane path: rows per work-item R (0 = 16).
VARIANTS = [0, 8, 32]


@pytest.mark.parametrize("k", VARIANTS)
@pytest.mark.parametrize("dtype", ["int32", "float32", "float64"])
@pytest.mark.parametrize("border,pad", [("pad", 0.0), ("pad", 1.0), ("nearest", 0.0)])
@pytest.mark.parametrize("shape", [(37, 20), (64, 64), (101, 300), (130, 1000)])
def test_bits_vs_oracle(dtype, border, pad, shape, k):
    x = grid(dtype, shape, seed=shape[0] * 7 + shape[1])
    for iters, tb, wc, wr in [(1, 1, 8, 8), (5, 2, 2, 16), (9, 4, 32, 8), (40, 33, 32, 8),
                              (12, 12, 1, 32), (7, 3, 3, 5)]:
        st, got = run_bits(x, iters, tb, wc, wr, border, pad, k=k)
        if got is None:
            continue
        want = oracle(st, x, iters)
        assert got.tobytes() == want.tobytes(), f"{dtype} {border}/{pad} {shape} it={iters} tb={tb} {wc}x{wr}"


@pytest.mark.parametrize("k", VARIANTS)
@pytest.mark.parametrize("tb", [1, 3, 31, 32, 33, 64, 100])
def test_bits_generation_counts(tb, k):
    x = grid("int32", (300, 520), seed=tb)
    for border in ("pad", "nearest"):
        st, got = run_bits(x, 100, tb, 32, 16, border, k=k)
        if got is not None:
            assert got.tobytes() == oracle(st, x, 100).tobytes(), f"tb={tb} {border}"


@pytest.mark.parametrize("wc,wr", [(1, 1), (2, 2), (4, 64), (32, 32), (64, 16), (512, 2),
                                   (7, 9), (100, 10)])
@pytest.mark.parametrize("k", [0, 8, 16, 32])
def test_bits_block_shapes(wc, wr, k):
    x = grid("int32", (257, 700), seed=wc * 31 + wr)
    try:
        st, got = run_bits(x, 20, 10, wc, wr, "nearest", k=k)
        if got is None:
            return
    except (RefusedParameter, IllegalWorkgroupSize):
        # a refusal must be the planned one: a tile too short for the halo
        # rows, or more threads than the kernel's register budget allows
        st = Stencil(op="gol", dtype="int32", border="nearest", load_path="bitplane",
                     fused_iterations=10, cells_per_thread=k)
        assert st.probe(700, 257, wc, wr)["status"] in ("REFUSED", "OVERSIZED")
        return
    assert got.tobytes() == oracle(st, x, 20).tobytes(), f"{wc}x{wr} K={k}"


def test_bits_config2_matches_per_cell_path():
    """BASELINE config 2 (8192^2, pad 0): 100 generations on the bit-plane path
    equal 100 single passes of the per-cell executor (a cheap full-size
    property; the oracle itself is checked at reduced size above)."""
    from paper_1511_02490_b200 import fill_host

    host = np.empty((8192, 8192), dtype=np.int32)
    fill_host(host, 2, 2)
    a = torch.from_numpy(host).cuda()
    ref = Stencil(op="gol", dtype="int32")
    want = ref.iterate(a.clone(), torch.empty_like(a), 100, 32, 8).clone()
    st = Stencil(op="gol", dtype="int32", fused_iterations=32)
    got = st.iterate(a.clone(), torch.empty_like(a), 100, 32, 8)
    torch.cuda.synchronize()
    assert torch.equal(got, want)


def test_bits_halo_rows_match_full_grid():
    """A row shard with TB-deep halos advances TB generations exactly like the
    same rows of the undivided grid (the multi-GPU fused exchange relies on
    this)."""
    x = grid("int32", (200, 333), seed=3)
    tb = 6
    for border, k in (("pad", 0), ("nearest", 0), ("pad", 8), ("nearest", 32)):
        st = Stencil(op="gol", dtype="int32", border=border, fused_iterations=tb,
                     load_path="bitplane", cells_per_thread=k)
        want = oracle(st, x, tb)
        for r0, r1 in [(0, 70), (70, 150), (150, 200), (3, 5)]:
            above, below = min(tb, r0), min(tb, 200 - r1)
            win = torch.from_numpy(np.ascontiguousarray(x[r0 - above:r1 + below])).cuda()
            out = torch.zeros((r1 - r0, 333), dtype=torch.int32, device="cuda")
            st(win[above:], out, 32, 8, rows_above=above, rows_below=below, height=r1 - r0)
            torch.cuda.synchronize()
            assert out.cpu().numpy().tobytes() == want[r0:r1].tobytes(), f"{border} rows {r0}:{r1}"


def test_bits_legality():
    st = Stencil(op="gol", dtype="int32", fused_iterations=32, load_path="bitplane")
    assert st.probe(8192, 8192, 32, 8)["load_path"] == "bitplane"
    km = st.kernel_max()
    assert km < 1024  # register-bound per-kernel maximum (R = 16 rows per lane)
    assert st.probe(8192, 8192, 32, 32)["status"] == "OVERSIZED"
    a = torch.zeros((64, 64), dtype=torch.int32, device="cuda")
    with pytest.raises(IllegalWorkgroupSize):
        st(a, torch.empty_like(a), 32, 32)
    # 8 warps x 8 rows per lane = a 64-row tile: no room for 2 x 32 halo rows
    big = Stencil(op="gol", dtype="int32", fused_iterations=32, load_path="bitplane",
                  cells_per_thread=8)
    assert big.probe(4096, 4096, 32, 8)["status"] == "REFUSED"
    with pytest.raises(RefusedParameter):
        big(a, torch.empty_like(a), 32, 8)
    with pytest.raises(Exception):
        Stencil(op="heat", dtype="float32", load_path="bitplane")(
            torch.zeros((8, 8), device="cuda"), torch.zeros((8, 8), device="cuda"), 8, 8)
