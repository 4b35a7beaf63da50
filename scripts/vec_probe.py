"""Scalar-TMA vs vector work-items: per-pass time over a block-size sweep for
the BASELINE workloads (gol 8192^2 i32, heat 16384^2 f32, boxmean (5,1,3,0)
4096^2 f32).  Prints one JSON line per (workload, path) with the best block,
its time and the HBM fraction (8 B/cell algorithmic)."""
from __future__ import annotations

import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1511_02490_b200 import RefusedParameter, IllegalWorkgroupSize, Stencil  # noqa: E402
from paper_1511_02490_b200._native import NativeError  # noqa: E402

PEAK = 6448.7
try:
    PEAK = float(json.loads((Path(__file__).resolve().parent.parent / "MEASURED_PEAKS.json").read_text())["hbm_gbs"])
except Exception:
    pass

WORK = {
    "gol": (dict(op="gol", dtype="int32"), 8192, 8192, torch.int32),
    "heat": (dict(op="heat", dtype="float32", border="nearest"), 16384, 16384, torch.float32),
    "boxmean": (dict(op="boxmean", dtype="float32", north=5, south=1, east=3, west=0, border="nearest"),
                4096, 4096, torch.float32),
}
SIZES = [(wc, wr) for wc in (2, 4, 8, 16, 24, 32, 48, 60, 64, 96, 128, 256) for wr in (1, 2, 4, 8, 16, 32)
         if wc * wr <= 1024 and wc * wr >= 32]

names = sys.argv[1:] or list(WORK)
for name in names:
    kw, W, H, tdt = WORK[name]
    a = (torch.rand((H, W), device="cuda") < 0.5).to(tdt) if tdt == torch.int32 else torch.rand((H, W), device="cuda")
    b = torch.empty_like(a)
    for path in ("tma", "vector"):
        st = Stencil(load_path=path, **kw)
        res = []
        for wc, wr in SIZES:
            try:
                ms = st.time(a, b, wc, wr, samples=10, warmup=2, flush_l2=True)
            except (RefusedParameter, IllegalWorkgroupSize, NativeError):
                continue
            res.append((sum(ms) / len(ms), wc, wr))
        res.sort()
        t, wc, wr = res[0]
        gbs = W * H * 8 / (t / 1e3) / 1e9
        print(json.dumps({"workload": name, "path": path, "best": f"{wc}x{wr}", "ms": round(t, 5),
                          "gcells": round(W * H / t / 1e6, 1), "hbm_frac": round(gbs / PEAK, 4),
                          "top5": [(f"{c}x{r}", round(x * 1e3, 2)) for x, c, r in res[:5]],
                          "sizes": len(res)}), flush=True)
