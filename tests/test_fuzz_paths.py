"""Property-based parity (hypothesis) of every execution path against the CPU
oracle: random op, element type, asymmetric borders, border mode / pad value,
grid shape (including 1-row / 1-column grids and shapes that are not
multiples of any tile), workgroup shape, cells per work-item, load path,
generations per launch and iteration count.  A configuration the executor
refuses, reports oversized or (for a forced load path the buffer cannot use)
reports ENOTSUP is fine; any executed configuration must be
bit-identical to the oracle.  Degenerate calls (zero-sized grids, negative
iterations, null buffers) must fail with EINVAL, never launch."""
from __future__ import annotations

import ctypes

import numpy as np
import pytest

import oracle_lib as O

torch = pytest.importorskip("torch")
hyp = pytest.importorskip("hypothesis")
from hypothesis import HealthCheck, given, settings  # noqa: E402
from hypothesis import strategies as st  # noqa: E402

pytestmark = pytest.mark.gpu

from paper_1511_02490_b200 import IllegalWorkgroupSize, RefusedParameter, Stencil  # noqa: E402
from paper_1511_02490_b200 import _native as N  # noqa: E402

TDT = {"int32": torch.int32, "float32": torch.float32, "float64": torch.float64}
SETTINGS = settings(max_examples=400, deadline=None, derandomize=True,
                    suppress_health_check=list(HealthCheck))


def make_grid(op, dtype, shape, seed):
    rng = np.random.default_rng(seed)
    if op == "gol":
        return (rng.random(shape) < 0.45).astype(dtype)
    if dtype == "int32":
        return rng.integers(-500, 500, size=shape).astype(np.int32)
    return (2 * rng.random(shape) - 1).astype(dtype)


def check(stc, x, iters, wc, wr):
    a = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    b = torch.empty_like(a)
    try:
        got = stc.iterate(a, b, iters, wc, wr)
    except (RefusedParameter, IllegalWorkgroupSize):
        return False
    except N.NativeError as exc:
        # a FORCED path may be impossible for the buffer (e.g. TMA needs 16-B
        # aligned rows): ENOTSUP, never a wrong result
        assert exc.code == N.SK_ENOTSUP and stc.load_path != "auto", str(exc)
        return False
    torch.cuda.synchronize()
    want = O.iterate(O.desc_from_stencil(stc), x, iters)
    assert got.cpu().numpy().tobytes() == want.tobytes(), repr(stc)
    return True


shapes = st.tuples(st.integers(1, 150), st.integers(1, 220))
blocks = st.tuples(st.integers(1, 64), st.integers(1, 16))


@SETTINGS
@given(op=st.sampled_from(["five_point", "heat", "gol", "boxmean", "sobel", "nms", "threshold",
                           "gaussian"]),
       dtype=st.sampled_from(["int32", "float32", "float64"]),
       borders=st.tuples(st.integers(0, 6), st.integers(0, 6), st.integers(0, 6), st.integers(0, 6)),
       nearest=st.booleans(), pad=st.sampled_from([0.0, 1.0, -2.5]), shape=shapes, block=blocks,
       k=st.sampled_from([0, 1, 2, 4, 8]), path=st.sampled_from(["auto", "tma", "explicit"]),
       iters=st.integers(1, 3), seed=st.integers(0, 10 ** 6))
def test_fuzz_one_pass_paths(op, dtype, borders, nearest, pad, shape, block, k, path, iters, seed):
    n, s, e, w = borders
    if op in ("five_point", "heat", "gol", "sobel", "nms"):
        n = s = e = w = 1
    elif op == "threshold":
        n = s = e = w = 0
    elif op == "gaussian":
        n = s = e = w = max(1, n)
    stc = Stencil(op=op, dtype=dtype, north=n, south=s, east=e, west=w,
                  border="nearest" if nearest else "pad", pad_value=pad, load_path=path,
                  cells_per_thread=k)
    check(stc, make_grid(op, dtype, shape, seed), iters, *block)


@SETTINGS
@given(kind=st.sampled_from(["fused", "bitplane", "strips"]),
       dtype=st.sampled_from(["int32", "float32", "float64"]), nearest=st.booleans(),
       pad=st.sampled_from([0.0, 1.0]), shape=shapes, block=blocks,
       tb=st.integers(1, 12), iters=st.integers(1, 30), kk=st.integers(0, 3), seed=st.integers(0, 10 ** 6))
def test_fuzz_temporal_paths(kind, dtype, nearest, pad, shape, block, tb, iters, kk, seed):
    if kind == "fused":
        op = ["heat", "five_point", "gol"][seed % 3]
        tb = 2 if tb % 2 else 4
        stc = Stencil(op=op, dtype=dtype, border="nearest" if nearest else "pad", pad_value=pad,
                      load_path="tma", fused_iterations=tb, cells_per_thread=[0, 1, 4, 8][kk])
    elif kind == "bitplane":
        op = "gol"
        stc = Stencil(op=op, dtype=dtype, border="nearest" if nearest else "pad", pad_value=pad,
                      load_path="bitplane", fused_iterations=tb, cells_per_thread=[0, 8, 16, 32][kk])
    else:
        op = ["heat", "five_point"][seed % 2]
        stc = Stencil(op=op, dtype=dtype, border="nearest" if nearest else "pad", pad_value=pad,
                      load_path="strips", fused_iterations=tb, cells_per_thread=[0, 4, 8, 16][kk])
    check(stc, make_grid(op, dtype, shape, seed), iters, *block)


def test_degenerate_calls_are_einval():
    stc = Stencil(op="heat", dtype="float32")
    a = torch.zeros((8, 8), device="cuda")
    lib = N.lib()
    in_b = ctypes.c_int32(0)
    for w, h, it in [(0, 8, 1), (8, 0, 1), (8, 8, -1)]:
        rc = lib.sk_stencil_iterate(ctypes.byref(stc.desc), a.data_ptr(), a.data_ptr(), w, h, 8, it, 8, 8,
                                    None, ctypes.byref(in_b))
        assert rc == N.SK_EINVAL, (w, h, it)
    rc = lib.sk_stencil_launch(ctypes.byref(stc.desc), None, a.data_ptr(), 8, 8, 8, 8, 0, 0, 8, 8, None)
    assert rc == N.SK_EINVAL
    # zero iterations leave the input untouched and report it in a
    assert lib.sk_stencil_iterate(ctypes.byref(stc.desc), a.data_ptr(), a.data_ptr(), 8, 8, 8, 0, 8, 8,
                                  None, ctypes.byref(in_b)) == N.SK_OK and in_b.value == 0


@settings(max_examples=60, deadline=None, derandomize=True, suppress_health_check=list(HealthCheck))
@given(op=st.sampled_from(["heat", "five_point", "gol", "boxmean", "sobel"]),
       dtype=st.sampled_from(["int32", "float32", "float64"]), world=st.integers(2, 4),
       rows_per_rank=st.integers(12, 40), width=st.integers(1, 200), nearest=st.booleans(),
       iters=st.integers(1, 9), calls=st.integers(1, 3), tb=st.sampled_from([0, 3, 6]),
       seed=st.integers(0, 10 ** 6))
def test_fuzz_peer_schedules(op, dtype, world, rows_per_rank, width, nearest, iters, calls, tb, seed):
    """Row shards on single-process ranks (one stream each) through
    sk_stencil_iterate_peer: one-generation schedule for every op, and the
    temporally blocked schedule (TB-deep halos) for heat / five_point."""
    from test_peer_halo import run_ranks

    n = s = e = w = 1
    if op == "boxmean":
        n, s, e, w = 5, 1, 3, 0
    fused = tb if op in ("heat", "five_point") else 0
    kw = {"load_path": "strips", "fused_iterations": fused} if fused else {}
    stc = Stencil(op=op, dtype=dtype, north=n, south=s, east=e, west=w,
                  border="nearest" if nearest else "pad", pad_value=0.5, **kw)
    x = make_grid(op, dtype, (world * rows_per_rank, width), seed)
    try:
        got = run_ranks(stc, x, world, iters, wc=32, wr=4, calls=min(calls, iters))
    except (RefusedParameter, IllegalWorkgroupSize):
        return
    except N.NativeError as exc:  # a shard too thin for TB-deep strips
        assert exc.code == N.SK_EINVAL and fused, str(exc)
        return
    want = O.iterate(O.desc_from_stencil(stc), x, iters)
    assert got.tobytes() == want.tobytes(), repr(stc)
