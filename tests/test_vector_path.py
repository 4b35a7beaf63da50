"""SK_LOAD_VECTOR (csrc/stencil/vector.cuh): vector work-items of 16 B of
cells x K rows, 128-bit shared loads and 128-bit global stores.  Bit-exact
against the CPU oracle for every op that has a vector form, every dtype,
both border modes, ragged grids (edge tiles in both directions) and a spread
of workgroup shapes; plus the refusal / not-supported contract."""
from __future__ import annotations

import numpy as np
import pytest

import oracle_lib as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_1511_02490_b200 import RefusedParameter, Stencil  # noqa: E402
from paper_1511_02490_b200 import _native as N  # noqa: E402

TDT = {"int32": torch.int32, "float32": torch.float32, "float64": torch.float64}


def grid(dtype, shape, seed, op):
    rng = np.random.default_rng(seed)
    if dtype == "int32":
        if op == "gol":
            return (rng.random(shape) < 0.45).astype(np.int32)
        return rng.integers(-1000, 1000, size=shape, dtype=np.int32)
    return (2 * rng.random(shape) - 1).astype(dtype)


def run(st: Stencil, x: np.ndarray, wc: int, wr: int, iters: int = 1) -> np.ndarray:
    a = torch.from_numpy(x).cuda()
    b = torch.empty_like(a)
    out = st.iterate(a, b, iters, wc, wr) if iters > 1 else (st(a, b, wc, wr), b)[1]
    torch.cuda.synchronize()
    return out.cpu().numpy()


OPS = [
    ("five_point", (1, 1, 1, 1)),
    ("heat", (1, 1, 1, 1)),
    ("gol", (1, 1, 1, 1)),
    ("sobel", (1, 1, 1, 1)),
    ("nms", (1, 1, 1, 1)),
    ("boxmean", (5, 1, 3, 0)),
]
SHAPES = [(2, 2), (4, 8), (8, 4), (16, 16), (32, 4), (2, 64), (24, 8), (60, 2), (6, 42)]


@pytest.mark.parametrize("dtype", ["int32", "float32", "float64"])
@pytest.mark.parametrize("border,pad", [("pad", 0.0), ("pad", 1.5), ("nearest", 0.0)])
@pytest.mark.parametrize("op,b", OPS)
def test_vector_matches_oracle(op, b, dtype, border, pad):
    if op == "gol" and border == "pad" and pad != 0.0:
        pad = 1.0
    st = Stencil(op=op, dtype=dtype, north=b[0], south=b[1], east=b[2], west=b[3], border=border,
                 pad_value=pad, load_path="vector")
    # 16-B aligned rows (pitch = W) with a width that is not a multiple of
    # any tile: edge tiles on the east and south sides of every shape
    x = grid(dtype, (203, 264), 7, op)
    want = O.stencil(O.desc_from_stencil(st), x)
    for wc, wr in SHAPES:
        got = run(st, x, wc, wr)
        assert got.tobytes() == want.tobytes(), f"{op} {dtype} {border} {wc}x{wr}"


@pytest.mark.parametrize("op,b", OPS)
def test_vector_equals_scalar_path_iterated(op, b):
    """Ten generations on the vector path == ten on the scalar TMA path."""
    dtype = "int32" if op == "gol" else "float32"
    x = grid(dtype, (300, 520), 11, op)
    kw = dict(op=op, dtype=dtype, north=b[0], south=b[1], east=b[2], west=b[3], border="nearest")
    got = run(Stencil(load_path="vector", **kw), x, 16, 8, iters=10)
    want = run(Stencil(load_path="tma", **kw), x, 32, 8, iters=10)
    assert got.tobytes() == want.tobytes()


def test_vector_gol_full_size_against_oracle():
    """BASELINE configs[1] grid on the vector path: 3 generations, bit-exact."""
    st = Stencil(op="gol", dtype="int32", load_path="vector")
    x = O.fill((8192, 8192), "int32", 2, 2)
    want = O.iterate(O.desc_from_stencil(st), x, 3)
    assert run(st, x, 32, 8, iters=3).tobytes() == want.tobytes()


def test_vector_boxmean_config4_against_oracle():
    """BASELINE configs[3] (4096^2 f32, (5,1,3,0), nearest) at a few blocks."""
    st = Stencil(op="boxmean", dtype="float32", north=5, south=1, east=3, west=0, border="nearest",
                 load_path="vector")
    x = O.fill((4096, 4096), "float32", 0, 4)
    want = O.stencil(O.desc_from_stencil(st), x)
    for wc, wr in [(24, 4), (32, 4), (16, 8), (8, 16), (2, 2)]:
        assert run(st, x, wc, wr).tobytes() == want.tobytes(), f"{wc}x{wr}"


def test_vector_contract():
    # no vector form: generic boxmean extents, gaussian, synthetic
    st = Stencil(op="boxmean", dtype="float32", north=2, south=2, east=2, west=2, load_path="vector")
    x = torch.zeros((64, 64), device="cuda")
    with pytest.raises(N.NativeError) as e:
        st(x, torch.empty_like(x), 8, 8)
    assert e.value.code == N.SK_ENOTSUP
    # wider than one TMA box (4 * 64 + 2 > 256 columns): refused, and the probe agrees
    st = Stencil(op="heat", dtype="float32", load_path="vector")
    x = torch.zeros((256, 1024), device="cuda")
    with pytest.raises(RefusedParameter):
        st(x, torch.empty_like(x), 64, 2)
    assert st.probe(1024, 256, 64, 2)["status"] == "REFUSED"
    assert st.probe(1024, 256, 32, 2)["load_path"] == "vector"
    # fused generations are not a vector-path feature
    with pytest.raises(N.NativeError) as e:
        Stencil(op="heat", dtype="float32", load_path="vector", fused_iterations=2)(
            x, torch.empty_like(x), 32, 2)
    assert e.value.code == N.SK_ENOTSUP
    # misaligned output pitch: not a vector-path buffer
    y = torch.zeros((256, 1025), device="cuda")
    with pytest.raises(N.NativeError) as e:
        st(x, y[:, 1:], 32, 2)
    assert e.value.code == N.SK_ENOTSUP
    # aligned pitch, output base 4 B off: the 16-B row stores are rejected ...
    flat = torch.zeros(256 * 1024 + 4, device="cuda")
    y = flat[1:1 + 256 * 1024].view(256, 1024)
    with pytest.raises(N.NativeError) as e:
        st(x, y, 32, 2)
    assert e.value.code == N.SK_EINVAL
    # ... while AUTO falls back to the scalar TMA kernel for that output
    x.uniform_()
    Stencil(op="heat", dtype="float32")(x, y, 32, 2)
    want = torch.empty_like(x)
    Stencil(op="heat", dtype="float32", load_path="tma")(x, want, 32, 2)
    torch.cuda.synchronize()
    assert torch.equal(y, want)
