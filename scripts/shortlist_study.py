"""Offline study of the measured shortlist (wgtb predict --shortlist N):
for every real-kernel scenario of the 30-observation re-sweep, the fastest
(by the recorded mean) of the model's N-size shortlist against the oracle.
N = 1 is the plain Algorithm-1 prediction.  In-sample with the all-scenario
bundle; held out with the leave-one-kernel-out bundles (gol, he).
usage: python scripts/shortlist_study.py [N ...]"""
import collections
import lzma
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
B = ROOT / "results" / "b200"
WGTB = ROOT / "paper_1511_02490_b200" / "lib" / "wgtb"
ns = [int(x) for x in sys.argv[1:]] or [1, 2, 4, 8]

runs = collections.defaultdict(lambda: collections.defaultdict(list))
with lzma.open(B / "real30" / "samples_real30.csv.xz", "rt") as f:
    next(f)
    for line in f:
        s, c, r, t = line.rstrip().split(",")
        runs[s][(int(c), int(r))].append(float(t))


def shortlist(model, kernel, ds, n):
    out = subprocess.run([str(WGTB), "predict", "--model", str(model), "--device", f"json:{B / 'device.json'}",
                          "--kernel-json", str(B / "descriptors" / "kernels" / f"{kernel}.json"),
                          "--dataset", ds, "--shortlist", str(n)], capture_output=True, text=True, check=True)
    v = list(map(int, out.stdout.split()))
    return list(zip(v[0::2], v[1::2]))


def study(model, kernels=None):
    perf = {n: [] for n in ns}
    for s in sorted(runs):
        _, k, size, types = s.split("/")
        if kernels and k not in kernels:
            continue
        mean = {w: sum(v) / len(v) for w, v in runs[s].items()}
        best = min(mean.values())
        sl = shortlist(model, k, f"{size}-{types}", max(ns))
        for n in ns:
            perf[n].append(best / min(mean[w] for w in sl[:n]))
    return {n: (sum(v) / len(v), min(v), len(v)) for n, v in perf.items()}


def show(label, res):
    print(label)
    for n, (m, lo, c) in res.items():
        print(f"  N={n:2d}: mean {100 * m:.1f} % of oracle, worst {100 * lo:.1f} % ({c} scenarios)")


show("in-sample, all-scenario bundle (results/b200/model.json), 136 real scenarios", study(B / "model.json"))
for k in ("gol", "he"):
    show(f"held out: {k} scenarios, bundle without {k} (model_loko_{k}.json)", study(B / f"model_loko_{k}.json", {k}))
