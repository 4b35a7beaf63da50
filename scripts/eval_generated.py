"""The executable study: the 40 GENERATED synthetic kernels
of the study (wgtb gen-kernel, swept by scripts/sweep_generated.py into
results/generated_r02) plus the 8 reference/BASELINE kernels from the
30-observation re-sweep (results/b200/real30), on the fp32 datasets
512^2 .. 8192^2.  Every kernel's code matches its descriptor.  Two descriptor
trees over the same samples - the reference's fixture instruction counts,
and counts binned from the SASS of the kernel that actually ran (generated
functor / built-in executor, scripts/sass_features.py) - and `wgtb evaluate`
on both (forest, tree, speedup regressor; 10-fold, synthetic->real,
leave-one-kernel-out).
usage: python scripts/eval_generated.py [OUT_DIR]"""
import importlib.util
import json
import lzma
import shutil
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
GEN = ROOT / "results" / "generated"
GEN2 = ROOT / "results" / "generated_r02"
B200 = ROOT / "results" / "b200"
WGTB = ROOT / "paper_1511_02490_b200" / "lib" / "wgtb"
spec = importlib.util.spec_from_file_location("sf", ROOT / "scripts" / "sass_features.py")
sf = importlib.util.module_from_spec(spec)
spec.loader.exec_module(sf)

SIDES = (512, 1024, 2048, 4096, 8192)
DATASETS = [f"{s}x{s}-FLOAT32-FLOAT32.json" for s in SIDES]
KEEP = tuple(f"/{s}x{s}/FLOAT32-FLOAT32" for s in SIDES)


def tree(dst: Path, sass: bool, swept: set):
    if dst.exists():
        shutil.rmtree(dst)
    (dst / "kernels").mkdir(parents=True)
    (dst / "datasets").mkdir()
    shutil.copytree(B200 / "descriptors" / "devices", dst / "devices")
    for ds in DATASETS:
        shutil.copy(B200 / "descriptors" / "datasets" / ds, dst / "datasets" / ds)
    for p in sorted((B200 / "descriptors" / "kernels").glob("*.json")):
        k = json.loads(p.read_text())
        if k["name"] not in swept:
            continue
        if sass:
            if k["name"].startswith("synthetic-"):
                funcs = sf.sass_functions(GEN / "lib" / f"lib{k['name']}.so")
                t = [n for n in funcs if "k_stencil_tma<wgtb::detail::UserOp<" in n and ", float, 8, 1024" in n]
                c = sf.categorise(funcs[t[0]])
                k["instr_counts"], k["total_instructions"] = c, sum(c.values())
            else:
                k = json.loads((B200 / "descriptors_sass" / "kernels" / p.name).read_text())
        (dst / "kernels" / p.name).write_text(json.dumps(k, indent=2, sort_keys=True) + "\n")


def lines(p: Path):
    with lzma.open(p, "rt") as f:
        yield from f


def samples(out: Path) -> set:
    out.mkdir(parents=True, exist_ok=True)
    swept = set()
    for name, gen_file, real_file in (("samples", "samples.csv.xz", "samples_real30.csv.xz"),
                                      ("refused", "refused.csv.xz", "refused_real30.csv.xz"),
                                      ("contexts", "contexts.csv.xz", "contexts_real30.csv.xz")):
        with open(out / f"{name}.csv", "w") as o:
            for k, ln in enumerate(lines(GEN2 / gen_file)):
                if k == 0 or ln.strip():
                    o.write(ln)
                    if name == "contexts" and k:
                        swept.add(ln.split("/")[1])
            for k, ln in enumerate(lines(B200 / "real30" / real_file)):
                sid = ln.split(",", 1)[0]
                if k and sid.endswith(KEEP):
                    o.write(ln)
                    if name == "contexts":
                        swept.add(sid.split("/")[1])
    return swept


def main():
    out = Path(sys.argv[1]) if len(sys.argv) > 1 else Path("/tmp/eval_generated")
    swept = samples(out)
    tree(out / "descriptors_fixture", False, swept)
    tree(out / "descriptors_sass", True, swept)
    rows = []
    for feats in ("fixture", "sass"):
        for part in ("kfold", "synthreal", "loo-kernel"):
            for tech in ("forest-nn", "tree-nn", "speedup-reg"):
                r = subprocess.run([str(WGTB), "evaluate", "--scenarios", str(out / f"descriptors_{feats}"),
                                    "--samples", str(out / "samples.csv"), "--refused", str(out / "refused.csv"),
                                    "--contexts", str(out / "contexts.csv"), "--technique", tech,
                                    "--partition", part], capture_output=True, text=True, check=True).stdout
                line = [ln for ln in r.splitlines() if ln.startswith(tech)][0].split()
                rows.append(f"{feats},{part},{tech},{line[1]},{line[4]}")
                print(rows[-1], flush=True)
    (GEN2 / "eval_features.csv").write_text("features,partition,technique,scenarios,perf_pct_oracle\n"
                                            + "\n".join(rows) + "\n")


if __name__ == "__main__":
    sys.exit(main())
