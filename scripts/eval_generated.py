"""Fixture vs SASS-derived kernel features on kernels whose code matches
their descriptors: the 16 generated synthetic kernels
(scripts/sweep_generated.py) plus the 6 reference kernels, fp32 datasets
512^2 .. 4096^2.  Builds two descriptor trees over the same samples - the
reference's fixture instruction counts, and counts binned from the SASS of
the kernel that actually ran (generated functor / built-in executor) - and
runs `wgtb evaluate` on both.
usage: python scripts/eval_generated.py"""
import importlib.util
import json
import shutil
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
GEN = ROOT / "results" / "generated"
B200 = ROOT / "results" / "b200"
WGTB = ROOT / "paper_1511_02490_b200" / "lib" / "wgtb"
spec = importlib.util.spec_from_file_location("sf", ROOT / "scripts" / "sass_features.py")
sf = importlib.util.module_from_spec(spec)
spec.loader.exec_module(sf)

DATASETS = [f"{s}x{s}-FLOAT32-FLOAT32.json" for s in (512, 1024, 2048, 4096)]
REAL = ["gaussian", "gol", "he", "nms", "sobel", "threshold"]


def tree(dst: Path, sass: bool):
    if dst.exists():
        shutil.rmtree(dst)
    (dst / "kernels").mkdir(parents=True)
    (dst / "datasets").mkdir()
    shutil.copytree(B200 / "descriptors" / "devices", dst / "devices")
    for ds in DATASETS:
        shutil.copy(B200 / "descriptors" / "datasets" / ds, dst / "datasets" / ds)
    src_sass = B200 / "descriptors_sass" / "kernels"
    for p in sorted((B200 / "descriptors" / "kernels").glob("*.json")):
        k = json.loads(p.read_text())
        if k["name"].startswith("synthetic-") and not (GEN / "lib" / f"lib{k['name']}.so").exists():
            continue  # only kernels that were generated (and swept) take part
        if sass:
            if k["name"].startswith("synthetic-"):
                funcs = sf.sass_functions(GEN / "lib" / f"lib{k['name']}.so")
                t = [n for n in funcs if "k_stencil_tma<wgtb::detail::UserOp<" in n and ", float, 8, 1024" in n]
                c = sf.categorise(funcs[t[0]])
                k["instr_counts"], k["total_instructions"] = c, sum(c.values())
            else:
                k = json.loads((src_sass / p.name).read_text())
        (dst / "kernels" / p.name).write_text(json.dumps(k, indent=2, sort_keys=True) + "\n")


def samples():
    keep = {f"/{s}x{s}/FLOAT32-FLOAT32" for s in (512, 1024, 2048, 4096)}
    lines = (GEN / "samples.csv").read_text().splitlines()
    ctx = (GEN / "contexts.csv").read_text().splitlines()
    ref = (GEN / "refused.csv").read_text().splitlines()
    for line in (B200 / "samples.csv").read_text().splitlines()[1:]:
        sid = line.split(",")[0]
        if sid.split("/")[1] in REAL and any(sid.endswith(k) for k in keep):
            lines.append(line)
    for line in (B200 / "contexts.csv").read_text().splitlines()[1:]:
        sid = line.split(",")[0]
        if sid.split("/")[1] in REAL and any(sid.endswith(k) for k in keep):
            ctx.append(line)
    for line in (B200 / "refused.csv").read_text().splitlines()[1:]:
        sid = line.split(",")[0]
        if sid.split("/")[1] in REAL and any(sid.endswith(k) for k in keep):
            ref.append(line)
    out = GEN / "eval"
    out.mkdir(exist_ok=True)
    (out / "samples.csv").write_text("\n".join(lines) + "\n")
    (out / "contexts.csv").write_text("\n".join(ctx) + "\n")
    (out / "refused.csv").write_text("\n".join(ref) + "\n")
    return out


def main():
    ev = samples()
    tree(ev / "descriptors_fixture", False)
    tree(ev / "descriptors_sass", True)
    rows = []
    for feats in ("fixture", "sass"):
        for part in ("kfold", "synthreal", "loo-kernel"):
            for tech in ("forest-nn", "tree-nn", "speedup-reg"):
                r = subprocess.run([str(WGTB), "evaluate", "--scenarios", str(ev / f"descriptors_{feats}"),
                                    "--samples", str(ev / "samples.csv"), "--refused", str(ev / "refused.csv"),
                                    "--contexts", str(ev / "contexts.csv"), "--technique", tech,
                                    "--partition", part], capture_output=True, text=True, check=True).stdout
                line = [ln for ln in r.splitlines() if ln.startswith(tech)][0].split()
                rows.append(f"{feats},{part},{tech},{line[1]},{line[4]}")
                print(rows[-1], flush=True)
    (GEN / "eval_features.csv").write_text("features,partition,technique,scenarios,perf_pct_oracle\n"
                                           + "\n".join(rows) + "\n")


if __name__ == "__main__":
    sys.exit(main())
