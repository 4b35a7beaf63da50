"""Exhaustive correctness sweep against the CPU oracle (GPU): every scenario of
a descriptor directory x every workgroup size of enumerate_space(1024), one
launch each, output compared bit-for-bit with the oracle.  Inputs are the
sweep's own (sk_fill_host with the executor's kind/seed).  Prints one line per
mismatching (scenario, size) and a summary.

usage: python scripts/verify_sweep.py DESCRIPTOR_DIR [--max-side N] [--kernel NAME ...]
"""
import argparse
import json
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import numpy as np
import torch

import oracle_lib as O
from paper_1511_02490_b200 import IllegalWorkgroupSize, RefusedParameter, Stencil, fill_host

ap = argparse.ArgumentParser()
ap.add_argument("desc_dir")
ap.add_argument("--max-side", type=int, default=4096)
ap.add_argument("--kernel", action="append", default=[])
ap.add_argument("--seed", type=int, default=1)
ap.add_argument("--k", type=int, default=0)
args = ap.parse_args()
d = Path(args.desc_dir)
kernels = [json.loads(p.read_text()) for p in sorted((d / "kernels").glob("*.json"))]
datasets = [json.loads(p.read_text()) for p in sorted((d / "datasets").glob("*.json"))]
sizes = [(c, r) for c in range(2, 513, 2) for r in range(2, 1024 // c + 1, 2)]
TDT = {"INT32": torch.int32, "FLOAT32": torch.float32, "FLOAT64": torch.float64}
NDT = {"INT32": np.int32, "FLOAT32": np.float32, "FLOAT64": np.float64}
bad_total = checked = 0
for k in kernels:
    if args.kernel and k["name"] not in args.kernel:
        continue
    for ds in datasets:
        if ds["width"] > args.max_side:
            continue
        t = ds["in_type"]
        st = Stencil.from_kernel(k["name"], k["north"], k["south"], k["east"], k["west"],
                                 dtype=t.lower(), complexity=int(k["complexity"]),
                                 instructions=k["total_instructions"],
                                 border="pad" if k["name"] == "gol" else "nearest",
                                 cells_per_thread=args.k)
        H, W = ds["height"], ds["width"]
        x = np.empty((H, W), NDT[t])
        kind = (2 if k["name"] == "gol" else 3) if t == "INT32" else 0
        fill_host(x, kind, args.seed)
        want = torch.from_numpy(O.stencil(O.desc_from_stencil(st), x, threads=os.cpu_count() or 8)).cuda()
        a = torch.from_numpy(x).cuda()
        b = torch.empty_like(a)
        bad = []
        for wc, wr in sizes:
            try:
                st(a, b, wc, wr)
            except (IllegalWorkgroupSize, RefusedParameter):
                continue
            if not torch.equal(b, want):
                nbad = int((b != want).sum())
                bad.append((wc, wr, nbad, st.probe(W, H, wc, wr)))
            checked += 1
        torch.cuda.synchronize()
        sid = f"{k['name']}/{W}x{H}/{t}"
        for wc, wr, nbad, pr in bad:
            print(f"MISMATCH {sid} {wc}x{wr} cells={nbad} {pr}", flush=True)
        bad_total += len(bad)
        print(f"done {sid}: {len(bad)} mismatching sizes", flush=True)
print(f"SUMMARY checked={checked} mismatching={bad_total}", flush=True)
