"""GPU parity: the sm_100a executor vs the CPU oracle (and the numpy golden
fixtures), through the C-ABI.  Bit-exact for every dtype (fp32/fp64 are
compiled without FMA contraction on both sides); the north-star tolerance for
fp32 (1e-5 relative) is asserted as well so a contraction regression is
reported with its size."""
from __future__ import annotations

from pathlib import Path

import numpy as np
import pytest

import oracle_lib as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_1511_02490_b200 import IllegalWorkgroupSize, RefusedParameter, Stencil  # noqa: E402

GOLDEN = Path(__file__).resolve().parent / "golden" / "stencil_golden.npz"
TDT = {"int32": torch.int32, "float32": torch.float32, "float64": torch.float64}
FP32_RTOL = 1e-5


def to_dev(x: np.ndarray):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def gpu_pass(st: Stencil, x: np.ndarray, wc: int, wr: int) -> np.ndarray:
    a = to_dev(x)
    b = torch.empty_like(a)
    st(a, b, wc, wr)
    torch.cuda.synchronize()
    return b.cpu().numpy()


def assert_same(got: np.ndarray, want: np.ndarray, what: str):
    assert got.dtype == want.dtype
    if got.dtype == np.float32:
        np.testing.assert_allclose(got, want, rtol=FP32_RTOL, atol=1e-6, err_msg=what)
    assert got.tobytes() == want.tobytes(), f"{what}: not bit-identical to the oracle"


def rand_grid(dtype, shape, seed, op="x"):
    rng = np.random.default_rng(seed)
    if dtype == "int32":
        if op == "gol":
            return (rng.random(shape) < 0.45).astype(np.int32)
        return rng.integers(-1000, 1000, size=shape, dtype=np.int32)
    return (2 * rng.random(shape) - 1).astype(dtype)


SHAPES = [(2, 2), (4, 2), (2, 16), (32, 4), (64, 4), (16, 16), (30, 6), (128, 2), (256, 4),
          (6, 42), (512, 2)]
PATHS = ["tma", "explicit"]


@pytest.mark.parametrize("name", sorted({k.split("__")[0]
                                          for k in np.load(GOLDEN).files}))
@pytest.mark.parametrize("path", PATHS)
def test_golden_cases(name, path):
    z = np.load(GOLDEN)
    x, y = z[f"{name}__in"], z[f"{name}__out"]
    n, s, e, w, nearest, cx, ins = (int(v) for v in z[f"{name}__meta"])
    st = Stencil(op=str(z[f"{name}__op"]), dtype=str(x.dtype), north=n, south=s, east=e, west=w,
                 border="nearest" if nearest else "pad", pad_value=float(z[f"{name}__pad"][0]),
                 complexity=cx, instructions=ins, load_path=path)
    # x is 23x37: fp32 rows are 148 B (not 16-B aligned) -> pad the pitch for TMA.
    for wc, wr in [(4, 2), (8, 8), (32, 4), (2, 30)]:
        a = torch.zeros((x.shape[0], 40), dtype=TDT[str(x.dtype)], device="cuda")
        a[:, :x.shape[1]] = to_dev(x)
        b = torch.zeros_like(a)
        st(a[:, :x.shape[1]], b[:, :x.shape[1]], wc, wr)
        torch.cuda.synchronize()
        got = b[:, :x.shape[1]].cpu().numpy()
        assert_same(got, y, f"{name} {path} {wc}x{wr}")


CASES = [
    ("five_point", "float32", (1, 1, 1, 1), "pad", 0.0),
    ("five_point", "float32", (1, 1, 1, 1), "pad", 1.0),
    ("five_point", "float64", (1, 1, 1, 1), "nearest", 0.0),
    ("heat", "float32", (1, 1, 1, 1), "nearest", 0.0),
    ("gol", "int32", (1, 1, 1, 1), "pad", 0.0),
    ("gol", "int32", (1, 1, 1, 1), "nearest", 0.0),
    ("boxmean", "float32", (5, 1, 3, 0), "nearest", 0.0),
    ("boxmean", "int32", (7, 2, 0, 9), "pad", -3.0),
    ("gaussian", "float32", (5, 5, 5, 5), "nearest", 0.0),
    ("gaussian", "int32", (10, 10, 10, 10), "pad", 0.0),
    ("sobel", "float64", (1, 1, 1, 1), "nearest", 0.0),
    ("nms", "float32", (1, 1, 1, 1), "pad", 0.0),
    ("threshold", "int32", (0, 0, 0, 0), "pad", 0.0),
]


@pytest.mark.parametrize("op,dtype,borders,border,pad", CASES)
@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("k", [0, 1, 2, 4, 8])
def test_ops_vs_oracle_ragged(op, dtype, borders, border, pad, path, k):
    n, s, e, w = borders
    st = Stencil(op=op, dtype=dtype, north=n, south=s, east=e, west=w, border=border,
                 pad_value=pad, load_path=path, cells_per_thread=k)
    H, W = 203, 264  # ragged vs every block shape; W*4 B is 16-B aligned
    x = rand_grid(dtype, (H, W), 11, op)
    want = O.stencil(O.desc_from_stencil(st), x)
    for wc, wr in SHAPES:
        if wc + e + w > 256 and path == "tma":
            continue
        if st.probe(W, H, wc, wr)["status"] != "OK":
            continue  # tile too large for shared memory at this K
        got = gpu_pass(st, x, wc, wr)
        assert_same(got, want, f"{op}/{dtype}/{border} {path} {wc}x{wr}")


@pytest.mark.parametrize("dtype", ["float32", "float64", "int32"])
@pytest.mark.parametrize("cx,ins", [(0, 100), (1, 650)])
def test_synthetic_vs_oracle(dtype, cx, ins):
    st = Stencil(op="synthetic", dtype=dtype, north=17, south=3, east=30, west=1,
                 border="nearest", complexity=cx, instructions=ins)
    x = rand_grid(dtype, (97, 160), 5)
    want = O.stencil(O.desc_from_stencil(st), x)
    for wc, wr in [(32, 8), (2, 64), (96, 2), (16, 6)]:
        assert_same(gpu_pass(st, x, wc, wr), want, f"synthetic {dtype} {wc}x{wr}")


def test_gol_config2_bit_exact_iterated():
    # BASELINE config 2 at a size the oracle finishes in seconds: 100 generations.
    st = Stencil(op="gol", dtype="int32")
    x = rand_grid("int32", (512, 512), 2, "gol")
    want = O.iterate(O.desc_from_stencil(st), x, 100)
    a, b = to_dev(x), torch.empty((512, 512), dtype=torch.int32, device="cuda")
    res = st.iterate(a, b, 100, 32, 8)
    torch.cuda.synchronize()
    assert res.cpu().numpy().tobytes() == want.tobytes()


def test_gol_full_size_properties():
    # Full BASELINE config-2 size: 8192^2, 100 generations.  The CPU oracle is
    # too slow here, so check size-independent properties: two block shapes
    # and both load paths agree bit-for-bit, outputs are {0,1}, and a periodic
    # tiling of blinkers is reproduced exactly.
    n = 8192
    x = rand_grid("int32", (n, n), 2, "gol")
    outs = []
    for wc, wr, path in [(32, 8, "tma"), (64, 4, "explicit"), (128, 2, "tma")]:
        st = Stencil(op="gol", dtype="int32", load_path=path)
        a, b = to_dev(x), torch.empty((n, n), dtype=torch.int32, device="cuda")
        outs.append(st.iterate(a, b, 100, wc, wr).cpu().numpy())
    assert outs[0].tobytes() == outs[1].tobytes() == outs[2].tobytes()
    assert set(np.unique(outs[0])) <= {0, 1}
    # blinkers on a 5-periodic lattice away from the edges: period 2
    g = np.zeros((n, n), np.int32)
    g[8:n - 8:5, 9:n - 8:5] = 1
    g[8:n - 8:5, 10:n - 7:5] = 1
    g[8:n - 8:5, 11:n - 6:5] = 1
    st = Stencil(op="gol", dtype="int32")
    a, b = to_dev(g), torch.empty((n, n), dtype=torch.int32, device="cuda")
    assert st.iterate(a, b, 100, 32, 8).cpu().numpy().tobytes() == g.tobytes()


def test_heat_config3_subset_iterated():
    st = Stencil(op="heat", dtype="float32", border="nearest")
    x = rand_grid("float32", (300, 520), 3)
    want = O.iterate(O.desc_from_stencil(st), x, 10)
    a, b = to_dev(x), torch.empty_like(to_dev(x))
    got = st.iterate(a, b, 10, 64, 4).cpu().numpy()
    assert_same(got, want, "heat x10")


def test_halo_rows_match_full_grid():
    st = Stencil(op="boxmean", dtype="float32", north=3, south=2, east=1, west=2,
                 border="nearest")
    x = rand_grid("float32", (64, 96), 9)
    full = gpu_pass(st, x, 32, 4)
    for path in PATHS:
        st2 = Stencil(op="boxmean", dtype="float32", north=3, south=2, east=1, west=2,
                      border="nearest", load_path=path)
        r0, r1 = 20, 41
        shard = to_dev(x[r0 - 3:r1 + 2])
        out = torch.empty((r1 - r0, 96), dtype=torch.float32, device="cuda")
        st2(shard[3:], out, 16, 8, rows_above=3, rows_below=2, height=r1 - r0)
        torch.cuda.synchronize()
        assert out.cpu().numpy().tobytes() == full[r0:r1].tobytes()


def test_oversized_and_refused():
    st = Stencil(op="gol", dtype="int32")
    a = torch.zeros((64, 64), dtype=torch.int32, device="cuda")
    b = torch.zeros_like(a)
    with pytest.raises(IllegalWorkgroupSize):
        st(a, b, 64, 32)  # 2048 threads
    assert st.probe(64, 64, 64, 32)["status"] == "OVERSIZED"
    # border 64 in f64 with a 512x2 block: tile (512+128)x(2+128)x8 B > 227 KB
    big = Stencil(op="boxmean", dtype="float64", north=64, south=64, east=64, west=64)
    assert big.probe(4096, 4096, 512, 2)["status"] == "REFUSED"
    a64 = torch.zeros((256, 1024), dtype=torch.float64, device="cuda")
    with pytest.raises(RefusedParameter) as ei:
        big(a64, torch.zeros_like(a64), 512, 2)
    assert (ei.value.w_c, ei.value.w_r) == (512, 2)
    # the context is still usable after a refusal
    st(a, b, 32, 8)
    torch.cuda.synchronize()


def test_kernel_max_and_probe_fields():
    st = Stencil(op="five_point", dtype="float32", cells_per_thread=1)
    km = st.kernel_max()
    assert 64 <= km <= 1024
    # AUTO takes 16-B vector work-items (4 fp32 cells per row) when the tile fits one TMA box
    p = st.probe(1024, 1024, 32, 8)
    assert p["status"] == "OK" and p["load_path"] == "vector"
    assert p["tile_bytes"] == (4 * 32 + 2) * (8 + 2) * 4
    # ... and the scalar TMA kernel past 256 box columns (4 * 64 + 2)
    assert st.probe(1024, 1024, 64, 8)["load_path"] == "tma"
    ps = Stencil(op="five_point", dtype="float32", cells_per_thread=1, load_path="tma").probe(1024, 1024, 32, 8)
    assert ps["load_path"] == "tma" and ps["tile_bytes"] == (32 + 2) * (8 + 2) * 4
    p4 = Stencil(op="five_point", dtype="float32", cells_per_thread=4,
                 load_path="tma").probe(1024, 1024, 32, 8)
    assert p4["tile_bytes"] == (32 + 2) * (8 * 4 + 2) * 4


def test_timing_returns_positive_samples():
    st = Stencil(op="five_point", dtype="float32")
    a = to_dev(rand_grid("float32", (1024, 1024), 1))
    b = torch.empty_like(a)
    ms = st.time(a, b, 32, 8, samples=5, warmup=2)
    assert len(ms) == 5 and all(t > 0 for t in ms)


def test_copy_ceiling_copies_and_times():
    """sk_copy_time: both kinds copy the bytes exactly, timed under the same
    harness as sk_stencil_time; misaligned kernel copies are EINVAL."""
    from paper_1511_02490_b200 import NativeError, copy_time

    a = to_dev(rand_grid("float32", (1024, 1024), 7))
    for kind in ("kernel", "memcpy"):
        b = torch.zeros_like(a)
        ms = copy_time(a, b, samples=4, warmup=1, kind=kind)
        assert len(ms) == 4 and all(t > 0 for t in ms)
        assert torch.equal(a, b)
    with pytest.raises(NativeError):
        copy_time(a.view(-1)[1:-3], torch.empty_like(a).view(-1)[:-4], samples=1, kind="kernel")


def test_run_host_end_to_end():
    st = Stencil(op="gol", dtype="int32")
    x = rand_grid("int32", (256, 300), 4, "gol")
    out = np.empty_like(x)
    st.run_host(x, out, 7, 32, 4)
    want = O.iterate(O.desc_from_stencil(st), x, 7)
    assert out.tobytes() == want.tobytes()


@pytest.mark.parametrize("op,dtype,borders,border", [
    ("gol", "int32", (1, 1, 1, 1), "pad"),
    ("boxmean", "float32", (5, 1, 3, 0), "nearest"),
    ("gaussian", "float64", (2, 2, 2, 2), "pad"),
])
def test_every_legal_size_matches_gold_standard(op, dtype, borders, border):
    """The paper validated every workgroup size against a gold-standard output
    (PAPER.md:446-450); the reference spec dropped it.  Restored:
    all 1,466 sizes of enumerate_space(1024) on both load paths."""
    n, s, e, w = borders
    x = rand_grid(dtype, (300, 328), 8, op)
    st0 = Stencil(op=op, dtype=dtype, north=n, south=s, east=e, west=w, border=border)
    want = O.stencil(O.desc_from_stencil(st0), x)
    a = to_dev(x)
    outs = {}
    sizes = [(c, r) for c in range(2, 513, 2) for r in range(2, 1024 // c + 1, 2)]
    assert len(sizes) == 1466
    for path in PATHS:
        st = Stencil(op=op, dtype=dtype, north=n, south=s, east=e, west=w, border=border,
                     load_path="auto" if path == "tma" else "explicit")
        for wc, wr in sizes:
            b = torch.full_like(a, 7)
            st(a, b, wc, wr)
            outs[(path, wc, wr)] = b
        torch.cuda.synchronize()
    bad = [k for k, b in outs.items() if b.cpu().numpy().tobytes() != want.tobytes()]
    assert not bad, f"{len(bad)} sizes differ, e.g. {bad[:5]}"


FUSED_CASES = [
    ("gol", "int32", (1, 1, 1, 1), "pad", 0.0),
    ("heat", "float32", (1, 1, 1, 1), "nearest", 0.0),
    ("five_point", "float64", (1, 1, 1, 1), "pad", 1.0),
    ("boxmean", "float32", (3, 2, 1, 0), "nearest", 0.0),
    ("boxmean", "int32", (1, 2, 2, 1), "pad", 7.0),
]


@pytest.mark.parametrize("op,dtype,borders,border,pad", FUSED_CASES)
@pytest.mark.parametrize("tb", [2, 4])
@pytest.mark.parametrize("k", [0, 1, 8])
def test_fused_iterations_vs_oracle(op, dtype, borders, border, pad, tb, k):
    """Temporal blocking (TB generations per launch) must equal TB one-pass
    generations exactly, including the per-generation border semantics."""
    n, s, e, w = borders
    st = Stencil(op=op, dtype=dtype, north=n, south=s, east=e, west=w, border=border,
                 pad_value=pad, cells_per_thread=k, fused_iterations=tb)
    x = rand_grid(dtype, (157, 200), 21, op)
    iters = 2 * tb + 1  # fused launches + a one-pass remainder
    want = O.iterate(O.desc_from_stencil(st), x, iters)
    for wc, wr in [(32, 8), (16, 16), (64, 2), (6, 10), (128, 4)]:
        if st.probe(200, 157, wc, wr)["status"] != "OK":
            continue
        a, b = to_dev(x), torch.empty_like(to_dev(x))
        got = st.iterate(a, b, iters, wc, wr).cpu().numpy()
        assert_same(got, want, f"fused TB={tb} K={k} {op}/{dtype} {wc}x{wr}")


def test_fused_single_launch_advances_tb_generations():
    st = Stencil(op="gol", dtype="int32", fused_iterations=4)
    x = rand_grid("int32", (256, 256), 3, "gol")
    want = O.iterate(O.desc_from_stencil(st), x, 4)
    a = to_dev(x)
    b = torch.empty_like(a)
    st(a, b, 32, 8)
    torch.cuda.synchronize()
    assert b.cpu().numpy().tobytes() == want.tobytes()


def test_fused_unsupported_op_is_enotsup():
    from paper_1511_02490_b200 import NativeError
    st = Stencil(op="sobel", dtype="float32", fused_iterations=2)
    a = to_dev(rand_grid("float32", (64, 64), 1))
    with pytest.raises(NativeError):
        st(a, torch.empty_like(a), 32, 8)


def test_stage_release_race_regression():
    """Regression: the warp released its TMA ring stage (mbarrier arrive)
    before its shared-memory loads had returned, so a refill could overwrite
    cells still being read - 523/3000 runs wrong on this exact configuration
    (2-stage ring, K=2, refills on every tile).  The arrive now follows the
    stores, which consume every loaded value."""
    st = Stencil(op="heat", dtype="float32", border="nearest")
    x = rand_grid("float32", (2048, 2048), 1)
    want = to_dev(O.stencil(O.desc_from_stencil(st), x))
    a = to_dev(x)
    outs = [torch.empty_like(a) for _ in range(4)]
    bad = 0
    for i in range(600):
        b = outs[i % 4]
        st(a, b, 2, 32)
        if i % 4 == 3:
            bad += sum(int(not torch.equal(o, want)) for o in outs)
    assert bad == 0


def test_in_process_autotuner_prediction_is_legal():
    """wgtb_predict (the in-process daemon): the trained bundle proposes a
    size for an unseen scenario, probed live; the size must launch and give
    the oracle's output."""
    from paper_1511_02490_b200 import autotune
    root = Path(__file__).resolve().parent.parent / "results" / "b200"
    st = Stencil(op="gol", dtype="int32")
    r = autotune.predict(st, 3000, 2000, root / "descriptors" / "kernels" / "gol.json",
                         root / "model.json")
    assert r["wc"] * r["wr"] <= 1024 and r["probes"] >= 1
    x = rand_grid("int32", (2000, 3000), 4, "gol")
    assert_same(gpu_pass(st, x, r["wc"], r["wr"]), O.stencil(O.desc_from_stencil(st), x), "predicted")


@pytest.mark.gpu
def test_streamed_host_jobs_match_run_host():
    """sk_stencil_submit_host / sk_stencil_wait_host (three slots in flight)
    give the same bytes as sk_stencil_run_host, for interleaved jobs of
    different inputs, sizes and iteration counts."""
    import torch

    st = Stencil(op="heat", dtype="float32", border="nearest")
    rng = np.random.default_rng(4)
    jobs = [(rng.random((300, 257)).astype(np.float32), 7), (rng.random((64, 900)).astype(np.float32), 4),
            (rng.random((300, 257)).astype(np.float32), 1), (rng.random((5, 5)).astype(np.float32), 3),
            (rng.random((129, 40)).astype(np.float32), 2)]
    ins = [torch.from_numpy(x).pin_memory() for x, _ in jobs]
    outs = [torch.empty_like(t).pin_memory() for t in ins]
    tickets = []
    for (x, it), hi, ho in zip(jobs, ins, outs):
        if len(tickets) >= 3:
            st.wait_host(tickets[-3])
        tickets.append(st.submit_host(hi, ho, it, 32, 8))
    for t in tickets:
        st.wait_host(t)
    for (x, it), ho in zip(jobs, outs):
        want = np.empty_like(x)
        st.run_host(x, want, it, 32, 8)
        assert ho.numpy().tobytes() == want.tobytes()
        assert want.tobytes() == O.iterate(O.desc_from_stencil(st), x, it).tobytes()
    with pytest.raises(Exception):
        st.wait_host(10 ** 9)


@pytest.mark.gpu
@pytest.mark.parametrize("path,wc,wr", [("auto", 64, 4), ("explicit", 64, 4), ("vector", 16, 8),
                                        ("vector", 8, 2), ("vector", 32, 4)])
def test_boxmean_division_special_values(path, wc, wr):
    """Config-4 boxmean divides by 28 with the exact 3-instruction sequence
    (ops.cuh div_const_fast) and falls back to IEEE division for a
    work-item whose sums include zeros, subnormals, huge values or inf:
    both branches must equal the oracle's s / 28 bit for bit.  The vector
    kernel divides optimistically and re-runs such a work-item with the fp64
    form (vector.cuh vblock_boxmean_exact)."""
    import torch

    rng = np.random.default_rng(12)
    x = (rng.random((200, 300)) - 0.5).astype(np.float32)
    x[10:20, :] = 0.0
    x[30:40, :] = (rng.random((10, 300)) * 1e-40).astype(np.float32)   # subnormal sums
    x[50:52, 100:120] = np.float32(3e37)                               # beyond the fast range
    x[60, 7] = np.inf
    x[80:82, :] = -0.0
    st = Stencil(op="boxmean", dtype="float32", north=5, south=1, east=3, west=0,
                 border="nearest", load_path=path)
    a = torch.from_numpy(x).cuda()
    b = torch.empty_like(a)
    st(a, b, wc, wr)
    torch.cuda.synchronize()
    want = O.stencil(O.desc_from_stencil(st), x)
    assert b.cpu().numpy().tobytes() == want.tobytes()


@pytest.mark.gpu
def test_streamed_bitplane_gol_jobs_and_concurrent_streams():
    """the bit-plane path's packed grids used to be one
    buffer pair per (device, thread), shared by the three streamed job slots
    and by user streams.  Three bit-plane GoL jobs in flight, and two
    iterate() calls on different user streams from one thread, must each
    equal the CPU oracle."""
    import torch

    st = Stencil(op="gol", dtype="int32", load_path="bitplane", fused_iterations=8)
    rng = np.random.default_rng(21)
    jobs = [((rng.random((700, 1031)) < 0.45).astype(np.int32), 37) for _ in range(6)]
    ins = [torch.from_numpy(x).pin_memory() for x, _ in jobs]
    outs = [torch.empty_like(t).pin_memory() for t in ins]
    tickets = []
    for (x, it), hi, ho in zip(jobs, ins, outs):
        if len(tickets) >= 3:
            st.wait_host(tickets[-3])
        tickets.append(st.submit_host(hi, ho, it, 32, 8))
    for t in tickets:
        st.wait_host(t)
    for (x, it), ho in zip(jobs, outs):
        assert ho.numpy().tobytes() == O.iterate(O.desc_from_stencil(st), x, it).tobytes()
    # two user streams, launches interleaved from one thread
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    xs = [torch.from_numpy(x).cuda() for x, _ in jobs[:2]]
    torch.cuda.synchronize()
    res = []
    for x, s in zip(xs, (s1, s2)):
        with torch.cuda.stream(s):
            res.append(st.iterate(x, torch.empty_like(x), 45, 32, 8, stream=s))
    torch.cuda.synchronize()
    for (x, _), r in zip(jobs[:2], res):
        assert r.cpu().numpy().tobytes() == O.iterate(O.desc_from_stencil(st), x, 45).tobytes()


@pytest.mark.parametrize("op,dtype,tb,iters", [("gol", "int32", 0, 70), ("heat", "float32", 0, 9),
                                               ("five_point", "float64", 2, 131), ("gol", "int32", 4, 64)])
def test_iterate_graph_replay_matches_oracle(op, dtype, tb, iters):
    """sk_stencil_iterate replays a captured CUDA graph from the third
    identical call on (64-generation chunks + remainder): every call - direct,
    capturing, replayed - equals the oracle, and result_in_b stays right."""
    st = Stencil(op=op, dtype=dtype, border="nearest" if op != "gol" else "pad", fused_iterations=tb,
                 load_path="tma" if tb else "auto")
    x = rand_grid(dtype, (97, 130), 12, op)
    want = O.iterate(O.desc_from_stencil(st), x, iters)
    a = torch.zeros((97, 132), dtype=TDT[dtype], device="cuda")[:, :130]
    b = torch.zeros((97, 132), dtype=TDT[dtype], device="cuda")[:, :130]
    for call in range(5):
        a.copy_(to_dev(x))
        got = st.iterate(a, b, iters, 16, 4)
        torch.cuda.synchronize()
        assert got.cpu().numpy().tobytes() == want.tobytes(), f"call {call}"


@pytest.mark.parametrize("op,dtype,W,wc,wr,border", [
    ("heat", "float32", 16384, 56, 4, "nearest"),   # vector, tiles_x = 74 (divides the 148-SM grid)
    ("heat", "float32", 16384, 224, 4, "nearest"),  # scalar TMA, tiles_x = 74
    ("heat", "int32", 8192, 28, 8, "nearest"),      # vector, tiles_x = 74
    ("boxmean", "float32", 4096, 28, 8, "nearest"),  # vector, tiles_x = 37
    ("gol", "int32", 8192, 112, 2, "pad"),           # scalar TMA, tiles_x = 74, pad 0
])
def test_balanced_grid_matches_oracle(op, dtype, W, wc, wr, border):
    """Sizes whose tile-column count divides 148 x occupancy: the persistent
    grid is trimmed so edge columns rotate over every CTA (launch.cu
    balanced_grid).  Tall enough that each CTA runs several tiles."""
    kw = dict(north=5, south=1, east=3, west=0) if op == "boxmean" else {}
    st = Stencil(op=op, dtype=dtype, border=border, **kw)
    x = rand_grid(dtype, (96, W), 31, op)
    want = O.stencil(O.desc_from_stencil(st), x)
    assert_same(gpu_pass(st, x, wc, wr), want, f"{op} {W} at {wc}x{wr}")


@pytest.mark.parametrize("op,dtype,wc,wr,border", [
    ("heat", "float32", 48, 8, "nearest"),       # 2 blocks x 2 stages -> 1 block x 3 stages
    ("heat", "float32", 40, 8, "nearest"),
    ("five_point", "float32", 44, 8, "pad"),
    ("gol", "int32", 48, 8, "pad"),
])
def test_deep_ring_matches_oracle(op, dtype, wc, wr, border):
    """Launches the ring-depth rule reshapes (launch.cu make_plan: one block
    with a three-stage ring, lag 2): several tiles per CTA so the ring wraps."""
    st = Stencil(op=op, dtype=dtype, border=border)
    x = rand_grid(dtype, (520, 8192), 41, op)
    want = O.stencil(O.desc_from_stencil(st), x)
    assert_same(gpu_pass(st, x, wc, wr), want, f"{op} at {wc}x{wr}")
