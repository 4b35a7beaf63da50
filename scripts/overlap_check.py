"""Token-sequence overlap of the host tuner sources with the reference files of
the same role (runs only where /root/reference exists; not shipped, not used
by the product).  Comments are stripped; a repo token counts as overlapping
when it lies inside an 8-token run that also occurs in the reference file.
A control pair (files of different roles) calibrates the floor that C++
boilerplate alone produces.
usage: python scripts/overlap_check.py [k]"""
import re
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
HOST = ROOT / "paper_1511_02490_b200" / "csrc" / "host"
REF = Path("/root/reference/proj/src")
PAIRS = [("learn.cpp", "learn.cpp"), ("evaluation.cpp", "bench.cpp"), ("autotune.cpp", "tuner.cpp"),
         ("space.cpp", "space.cpp"), ("io.cpp", "datastore.cpp"), ("scenario.cpp", "synthgen.cpp")]
CONTROL = [("learn.cpp", "bench.cpp"), ("evaluation.cpp", "learn.cpp")]


def tokens(path):
    s = path.read_text()
    s = re.sub(r"//[^\n]*", "", s)
    s = re.sub(r"/\*.*?\*/", "", s, flags=re.S)
    return re.findall(r"[A-Za-z_]\w*|\d+|\S", s)


def overlap(a, b, k):
    ta, tb = tokens(a), tokens(b)
    grams = {tuple(tb[i:i + k]) for i in range(len(tb) - k + 1)}
    cov = [False] * len(ta)
    for i in range(len(ta) - k + 1):
        if tuple(ta[i:i + k]) in grams:
            cov[i:i + k] = [True] * k
    return sum(cov) / max(1, len(ta))


def main():
    k = int(sys.argv[1]) if len(sys.argv) > 1 else 8
    if not REF.exists():
        print("no /root/reference here")
        return
    for mine, ref in PAIRS:
        print(f"{mine:16s} vs {ref:14s} {overlap(HOST / mine, REF / ref, k):.3f}")
    for mine, ref in CONTROL:
        print(f"control {mine:8s} vs {ref:14s} {overlap(HOST / mine, REF / ref, k):.3f}")


if __name__ == "__main__":
    main()
