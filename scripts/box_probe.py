"""Config 4 (box mean (5,1,3,0), 4096^2 f32, nearest border): flushed
single-pass time at a few blocks x cells per work-item (K; 0 = AUTO), on
the vector path, with the size-matched copy ceiling beside it; and the
output checked against the CPU oracle once per (block, K).
usage: python scripts/box_probe.py [samples]"""
import json
import sys
from pathlib import Path

import os

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
if os.environ.get("VARIANT_ROOT"):  # an alternative build of the package (A/B experiments)
    sys.path.insert(0, os.environ["VARIANT_ROOT"])
sys.path.insert(0, str(ROOT / "tests"))
import numpy as np
import torch

import oracle_lib as O  # checker only
from paper_1511_02490_b200 import Stencil, copy_time

n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
H = W = 4096
x = (2 * np.random.default_rng(1).random((H, W), dtype=np.float32) - 1).astype(np.float32)
a = torch.from_numpy(x).cuda()
b = torch.empty_like(a)
want = O.stencil(O.desc_from("boxmean", "float32", 5, 1, 3, 0, "nearest"), x)
peak = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"]
nbytes = 2 * a.numel() * 4
out = {"copy_kernel_us": float(np.median(copy_time(a, b, samples=n, warmup=3, flush_l2=True, kind="kernel"))) * 1e3}
import paper_1511_02490_b200 as PKG

out["package"] = str(Path(PKG.__file__).parent)
blocks = [(16, 8), (32, 4), (16, 4), (8, 8), (32, 2), (24, 8), (16, 16)]
ks = (0, 4, 8, 16)
if os.environ.get("QUICK"):
    blocks, ks = [(16, 8), (32, 4), (8, 8), (16, 16)], (4, 8)
for wc, wr in blocks:
    for K in ks:
        st = Stencil(op="boxmean", dtype="float32", north=5, south=1, east=3, west=0, border="nearest",
                     load_path="vector", cells_per_thread=K)
        try:
            st(a, b, wc, wr)
            torch.cuda.synchronize()
            ok = b.cpu().numpy().tobytes() == want.tobytes()
            us = float(np.median(st.time(a, b, wc, wr, samples=n, warmup=3, flush_l2=True))) * 1e3
        except Exception as e:  # refused / unsupported
            out[f"{wc}x{wr} K{K}"] = str(e)[:60]
            continue
        out[f"{wc}x{wr} K{K}"] = {"us": round(us, 2), "frac": round(nbytes / (us * 1e-6) / 1e9 / peak, 4),
                                  "exact": ok}
print(json.dumps(out, indent=1))
