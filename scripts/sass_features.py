"""Kernel features from the compiled sm_100a code (the
static-count half): the paper counts instructions per category in the
kernel's LLVM IR; the reference replaces that with fixture
splits (src/synthgen.cpp:16-38, 89-94).  Here the counts come from the SASS
of the executor kernel that actually runs each KernelDescriptor
(k_stencil_tma<Op, float, 8, 1024>, cuobjdump), binned into the reference's
eight categories (scenario.hpp:24: load, store, int_arith, float_arith,
branch, vector, call, other).

Writes a descriptor tree with SASS-derived instr_counts / total_instructions
(devices/ and datasets/ copied unchanged; scenario ids are unchanged) and a
CSV comparing fixture and SASS densities.

usage: python scripts/sass_features.py [descriptors_in] [descriptors_out] [csv_out]"""
from __future__ import annotations

import collections
import json
import re
import shutil
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
OBJ = ROOT / "paper_1511_02490_b200" / "lib" / "kernels_f32.o"
CATS = ["load", "store", "int_arith", "float_arith", "branch", "vector", "call", "other"]

# SASS opcode (before the first '.') -> reference category
OPCODES = {
    "load": {"LDG", "LDS", "LD", "LDL", "LDC", "LDCU", "ULDC", "LDSM", "LDGSTS", "UTMALDG", "UBLKCP",
             "LDGDEPBAR"},
    "store": {"STG", "STS", "ST", "STL", "UTMASTG", "RED", "ATOM", "ATOMS", "ATOMG"},
    "int_arith": {"IMAD", "IADD3", "IADD", "LOP3", "LOP", "SHF", "SHL", "SHR", "LEA", "ISETP", "IMNMX",
                  "VIMNMX", "IABS", "POPC", "FLO", "BREV", "SEL", "VIADD", "IDP", "I2I", "IMUL",
                  "UIADD3", "UIMAD", "ULOP3", "UISETP", "ULEA", "USEL", "USHF", "UFLO", "UPOPC", "UIMNMX",
                  "UMOV", "UPRMT", "PRMT", "VIADDMNMX", "IMNMX3", "UBREV", "USGXT", "SGXT", "BMSK", "UBMSK"},
    "float_arith": {"FADD", "FMUL", "FFMA", "FADD2", "FMUL2", "FFMA2", "FSETP", "FMNMX", "MUFU", "FSEL",
                    "FCHK", "DADD", "DMUL", "DFMA", "DSETP", "DMNMX", "F2I", "I2F", "F2F", "FRND",
                    "HADD2", "HFMA2", "HMUL2", "I2FP", "F2IP", "FSWZADD", "DSEL"},
    "branch": {"BRA", "BRX", "JMP", "JMX", "EXIT", "BSSY", "BSYNC", "WARPSYNC", "BREAK", "KILL", "YIELD",
               "NANOSLEEP", "BPT"},
    "vector": {"SHFL", "VOTE", "VOTEU", "MATCH", "REDUX", "CREDUX"},
    "call": {"CALL", "RET"},
}
OP2CAT = {op: cat for cat, ops in OPCODES.items() for op in ops}

KERNEL_OP = {"gaussian": "GaussianFixed<5>", "gol": "Gol", "he": "Heat", "nms": "Nms",
             "sobel": "Sobel", "threshold": "Threshold", "five_point": "FivePoint",
             "boxmean-5130": "BoxMeanFixed<5, 1, 3, 0>"}


def sass_functions(obj: Path) -> dict[str, list[str]]:
    """demangled function name -> list of SASS opcodes"""
    text = subprocess.run(["cuobjdump", "-sass", str(obj)], capture_output=True, text=True,
                          check=True).stdout
    funcs, cur = {}, None
    for line in text.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            name = subprocess.run(["c++filt", m.group(1)], capture_output=True, text=True).stdout.strip()
            cur = funcs.setdefault(name, [])
            continue
        m = re.match(r"\s+/\*[0-9a-f]{4}\*/\s+(?:@!?U?P[0-9T]\s+)?([A-Z][A-Z0-9_]*)", line)
        if m and cur is not None:
            cur.append(m.group(1))
    return funcs


def categorise(ops: list[str]) -> dict[str, int]:
    c = collections.Counter(OP2CAT.get(op, "other") for op in ops if op != "NOP")
    return {k: int(c.get(k, 0)) for k in CATS}


def main() -> int:
    src = Path(sys.argv[1]) if len(sys.argv) > 1 else ROOT / "results" / "b200" / "descriptors"
    dst = Path(sys.argv[2]) if len(sys.argv) > 2 else ROOT / "results" / "b200" / "descriptors_sass"
    csv_out = Path(sys.argv[3]) if len(sys.argv) > 3 else ROOT / "results" / "b200" / "sass_features.csv"
    funcs = sass_functions(OBJ)

    def counts_for(op: str) -> dict[str, int]:
        # the kernel AUTO runs for fp32: the vector work-item instantiation
        # when the op has one (vector.cuh), else the scalar one-pass kernel
        vec = re.compile(rf"void sk::k_stencil_tma_r80<sk::{re.escape(op)}, float, 8, 4>\(")
        hits = [n for n in funcs if vec.match(n)]
        if hits:
            return categorise(funcs[hits[0]])
        want = re.compile(rf"void sk::k_stencil_tma<sk::{re.escape(op)}, float, 8, 1024(, false(, 1)?)?>\(")
        hits = [n for n in funcs if want.match(n)]
        if len(hits) != 1:
            raise SystemExit(f"no unique SASS function for {want}: {hits[:3]}")
        return categorise(funcs[hits[0]])

    if dst.exists():
        shutil.rmtree(dst)
    shutil.copytree(src / "devices", dst / "devices")
    shutil.copytree(src / "datasets", dst / "datasets")
    (dst / "kernels").mkdir(parents=True)
    rows = ["kernel,source," + ",".join(f"d_{c}" for c in CATS) + ",total"]
    for p in sorted((src / "kernels").glob("*.json")):
        k = json.loads(p.read_text())
        op = "Synthetic" if k["name"].startswith("synthetic-") else KERNEL_OP[k["name"]]
        sass = counts_for(op)
        tot_f, tot_s = k["total_instructions"], sum(sass.values())
        rows.append(f"{k['name']},fixture," + ",".join(f"{k['instr_counts'][c] / tot_f:.4f}" for c in CATS)
                    + f",{tot_f}")
        rows.append(f"{k['name']},sass:{op}," + ",".join(f"{sass[c] / tot_s:.4f}" for c in CATS)
                    + f",{tot_s}")
        k["instr_counts"] = sass
        k["total_instructions"] = tot_s
        (dst / "kernels" / p.name).write_text(json.dumps(k, indent=2, sort_keys=True) + "\n")
    csv_out.write_text("\n".join(rows) + "\n")
    print(f"wrote {dst} and {csv_out}")
    return 0


if __name__ == "__main__":
    sys.exit(main())
