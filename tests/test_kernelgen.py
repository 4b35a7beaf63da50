"""Executable synthetic kernels (include/wgtb/
kernelgen.hpp): `wgtb gen-kernel` turns a reference KernelDescriptor into a
CUDA customising function (template substitution) and a C reference of the
same computation.  CPU: generation is deterministic and the C reference
builds and runs.  GPU: the generated functor, built against the executor's
kernel templates and launched through sk_stencil_launch_custom, is bit-exact
to the C reference over both border modes, and its SASS profile follows the
descriptor (scripts/sass_features.py binning)."""
from __future__ import annotations

import ctypes
import importlib.util
import json
import shutil
import subprocess
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
WGTB = ROOT / "paper_1511_02490_b200" / "lib" / "wgtb"
KDIR = ROOT / "results" / "b200" / "descriptors" / "kernels"
NAMES = ["synthetic-17-0", "synthetic-17-3", "synthetic-17-11"]


def generate(name, out):
    subprocess.run([str(WGTB), "gen-kernel", "--kernel-json", str(KDIR / f"{name}.json"), "--out", str(out)],
                   check=True, capture_output=True, timeout=60)
    return out / f"{name}.cu", out / f"{name}_ref.c"


def build_ref(c_src, out):
    so = out / (c_src.stem + ".so")
    subprocess.run(["gcc", "-O2", "-ffp-contract=off", "-fPIC", "-shared", str(c_src), "-o", str(so)],
                   check=True, timeout=120)
    lib = ctypes.CDLL(str(so))
    lib.gen_grid.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_long, ctypes.c_long, ctypes.c_int,
                             ctypes.c_float]
    return lib


def ref_grid(lib, x, mode, pad):
    out = np.empty_like(x)
    lib.gen_grid(x.ctypes.data, out.ctypes.data, x.shape[1], x.shape[0], mode, pad)
    return out


@pytest.mark.skipif(not WGTB.exists() or not shutil.which("gcc"), reason="needs the built wgtb CLI")
def test_generation_is_deterministic_and_c_reference_runs(tmp_path):
    a, _ = generate(NAMES[0], tmp_path / "a")
    b, c = generate(NAMES[0], tmp_path / "b")
    assert a.read_text() == b.read_text()
    k = json.loads((KDIR / f"{NAMES[0]}.json").read_text())
    src = a.read_text()
    assert src.count("v.at(") == max(1, k["instr_counts"]["load"]) + 1  # taps + centre
    assert f"v.at({-k['north']}, 0)" in src and f"v.at(0, {k['east']})" in src
    lib = build_ref(c, tmp_path / "b")
    x = np.random.default_rng(0).random((40, 50)).astype(np.float32)
    y = ref_grid(lib, x, 1, 0.0)
    assert np.isfinite(y).all() and not np.array_equal(y, x)


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_generated_kernel_matches_c_reference(name, tmp_path):
    torch = pytest.importorskip("torch")
    from paper_1511_02490_b200 import _native as N

    cu, c = generate(name, tmp_path)
    so = tmp_path / f"lib{name}.so"
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++20", "-fmad=false",
                    "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC", "-shared",
                    "-I", str(ROOT / "include"), "-I", str(ROOT / "paper_1511_02490_b200" / "csrc" / "stencil"),
                    str(cu), "-o", str(so)], check=True, timeout=600)
    gen = ctypes.CDLL(str(so))
    table = (ctypes.c_void_p * 8)()
    assert gen.sk_gen_table(ctypes.byref(table)) == 0
    ref = build_ref(c, tmp_path)
    k = json.loads((KDIR / f"{name}.json").read_text())
    x = np.random.default_rng(len(name)).random((150, 260)).astype(np.float32)
    for mode, pad in ((1, 0.0), (0, 0.5)):
        d = N.sk_stencil_desc(op=0, dtype=N.SK_FLOAT32, north=k["north"], south=k["south"], east=k["east"],
                              west=k["west"], border_mode=mode, pad_value=pad)
        want = ref_grid(ref, x, mode, pad)
        for wc, wr in ((32, 8), (64, 4)):
            a = torch.from_numpy(x).cuda()
            b = torch.empty_like(a)
            rc = N.lib().sk_stencil_launch_custom(ctypes.byref(d), ctypes.byref(table), a.data_ptr(),
                                                  b.data_ptr(), 260, 150, 260, 260, 0, 0, wc, wr, None)
            if rc in (N.SK_REFUSED, N.SK_OVERSIZED):
                continue
            assert rc == 0, N.last_error()
            torch.cuda.synchronize()
            assert b.cpu().numpy().tobytes() == want.tobytes(), (name, mode, wc, wr)
    # the compiled functor's SASS follows the descriptor's mix
    spec = importlib.util.spec_from_file_location("sf", ROOT / "scripts" / "sass_features.py")
    sf = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(sf)
    funcs = sf.sass_functions(so)
    tma8 = [n for n in funcs if "k_stencil_tma<wgtb::detail::UserOp<" in n and ", float, 8, 1024" in n]
    assert len(tma8) == 1
    counts = sf.categorise(funcs[tma8[0]])
    assert counts["float_arith"] >= k["instr_counts"]["float_arith"] // 2
