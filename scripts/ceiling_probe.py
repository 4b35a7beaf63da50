"""Size-matched streaming ceilings (sk_copy_time) next to the one-pass
stencil at the BASELINE shapes: copy GB/s vs bytes, flushed and back to
back, and the stencil's fraction of each.  One JSON line per case.
usage: python scripts/ceiling_probe.py > gpurun_out/ceiling.jsonl"""
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1511_02490_b200 import Stencil, copy_time  # noqa: E402

peak = json.loads((Path(__file__).resolve().parent.parent / "MEASURED_PEAKS.json").read_text())
peak = float(peak.get("hbm_gbs") or peak.get("hbm_copy_gbs"))

for side in (1024, 2048, 4096, 8192, 16384):
    a = torch.rand(side, side, device="cuda")
    b = torch.empty_like(a)
    nbytes = 2 * a.numel() * 4
    for flushed in (True, False):
        for kind in ("kernel", "memcpy"):
            ms = float(np.median(copy_time(a, b, samples=30, warmup=3, flush_l2=flushed, kind=kind)))
            print(json.dumps({"side": side, "bytes": nbytes, "flushed": flushed, "kind": kind,
                              "us": round(ms * 1e3, 2), "gbs": round(nbytes / ms / 1e6, 1),
                              "frac_of_peak": round(nbytes / ms / 1e6 / peak, 4)}), flush=True)

cases = [("boxmean", dict(north=5, south=1, east=3, west=0, border="nearest"), 4096, (8, 8), True),
         ("heat", dict(border="nearest"), 16384, (88, 8), False),
         ("five_point", dict(), 1024, (32, 8), True)]
for op, kw, side, (wc, wr), flushed in cases:
    st = Stencil(op=op, dtype="float32", **kw)
    a = torch.rand(side, side, device="cuda")
    b = torch.empty_like(a)
    ms = float(np.median(st.time(a, b, wc, wr, samples=30, warmup=3, flush_l2=flushed)))
    cp = float(np.median(copy_time(a, b, samples=30, warmup=3, flush_l2=flushed, kind="kernel")))
    print(json.dumps({"op": op, "side": side, "block": f"{wc}x{wr}", "flushed": flushed,
                      "stencil_us": round(ms * 1e3, 2), "copy_us": round(cp * 1e3, 2),
                      "stencil_over_copy": round(cp / ms, 4),
                      "stencil_frac_of_peak": round(2 * side * side * 4 / ms / 1e6 / peak, 4)}), flush=True)
