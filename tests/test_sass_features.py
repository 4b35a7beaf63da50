"""SASS-derived kernel features (scripts/sass_features.py; SURVEY.md §8f
rank 3, static-count half): opcode binning into the reference's eight
instruction categories (scenario.hpp:24) and extraction from the built
sm_100a object.  CPU only (cuobjdump disassembles without a GPU)."""
from __future__ import annotations

import importlib.util
import re
import shutil
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
spec = importlib.util.spec_from_file_location("sass_features", ROOT / "scripts" / "sass_features.py")
sf = importlib.util.module_from_spec(spec)
spec.loader.exec_module(sf)


def test_categorise_bins_every_opcode_once():
    ops = ["LDS", "LDG", "STG", "IMAD", "LOP3", "FADD", "FFMA", "MUFU", "BRA", "EXIT", "SHFL", "CALL",
           "MOV", "S2R", "NOP", "BAR"]
    c = sf.categorise(ops)
    assert list(c) == sf.CATS
    assert c == {"load": 2, "store": 1, "int_arith": 2, "float_arith": 3, "branch": 2, "vector": 1,
                 "call": 1, "other": 3}  # NOP is not counted
    assert sum(c.values()) == len(ops) - 1


@pytest.mark.skipif(not shutil.which("cuobjdump") or not sf.OBJ.exists(), reason="needs cuobjdump + build")
def test_executor_kernels_have_sass_features():
    funcs = sf.sass_functions(sf.OBJ)
    def one(op):
        want = re.compile(rf"void sk::k_stencil_tma<sk::{op}, float, 8, 1024(, false(, 1)?)?>\(")
        hits = [n for n in funcs if want.match(n)]
        assert len(hits) == 1, op
        return sf.categorise(funcs[hits[0]])

    for op in ("Heat", "Gol", "Sobel", "Synthetic"):
        c = one(op)
        assert sum(c.values()) > 100 and c["load"] > 0 and c["store"] > 0 and c["branch"] > 0
    heat, gol = one("Heat"), one("Gol")
    assert heat["float_arith"] > gol["float_arith"]  # heat is FP work, gol counts integers
