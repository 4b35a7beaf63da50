"""Layer the round-2 30-observation re-sweep of the reference kernels
(results/b200/real30) over the round-1 study (results/b200: 662 scenarios,
5-sample means) into plain CSV files a single-file reader (the reference's
load_samples / ref_evaluate) can take: every scenario of the re-sweep
replaces the round-1 rows, refusals and context of that scenario.
usage: python scripts/merge_study.py OUT_DIR"""
import gzip
import lzma
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
B = ROOT / "results" / "b200"
out = Path(sys.argv[1])
out.mkdir(parents=True, exist_ok=True)


def lines(p: Path):
    op = gzip.open if p.suffix == ".gz" else lzma.open if p.suffix == ".xz" else open
    with op(p, "rt") as f:
        yield from f


new_ids = {ln.split(",", 1)[0] for i, ln in enumerate(lines(B / "real30" / "contexts_real30.csv.xz")) if i}
for name, old, new in [("samples.csv", B / "samples.csv.gz", B / "real30" / "samples_real30.csv.xz"),
                       ("refused.csv", B / "refused.csv", B / "real30" / "refused_real30.csv.xz"),
                       ("contexts.csv", B / "contexts.csv", B / "real30" / "contexts_real30.csv.xz")]:
    rows = []
    header = None
    for src, keep in ((old, lambda i: i not in new_ids), (new, lambda i: True)):
        for k, ln in enumerate(lines(src)):
            if k == 0:
                header = header or ln
                continue
            if ln.strip() and keep(ln.split(",", 1)[0]):
                rows.append(ln)
    rows.sort(key=lambda ln: ln.split(",", 1)[0])  # stable: groups stay contiguous, in order
    with open(out / name, "w") as f:
        f.write(header)
        f.writelines(rows)
    print(name, len(rows))
