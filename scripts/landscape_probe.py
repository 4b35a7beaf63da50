"""Per-size pass times over a slice of the wc x wr space for heat 16384^2,
GoL 8192^2 and the config-4 box mean (flushed single passes, median of N, us),
for A/B of launch-policy switches (run under different SK_* environments).
usage: python scripts/landscape_probe.py [samples]"""
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

from paper_1511_02490_b200 import Stencil

samples = int(sys.argv[1]) if len(sys.argv) > 1 else 7
cases = [
    (dict(op="heat", dtype="float32", border="nearest"), 16384,
     [(c, r) for r in (4, 6, 8, 16) for c in range(8, 64, 4)] + [(c, r) for r in (4, 8) for c in (88, 120, 160, 232)]),
    (dict(op="gol", dtype="int32"), 8192,
     [(c, r) for r in (4, 8, 16, 28) for c in range(8, 64, 8)] + [(128, 8), (256, 4)]),
    (dict(op="boxmean", dtype="float32", north=5, south=1, east=3, west=0, border="nearest"), 4096,
     [(c, r) for r in (2, 4, 8, 16) for c in range(4, 64, 4)] + [(96, 4), (128, 4)]),
]
out = {"env": {k: v for k, v in os.environ.items() if k.startswith("SK_")}}
for kw, n, sizes in cases:
    st = Stencil(**kw)
    a = torch.rand((n, n), device="cuda")
    if kw["dtype"] == "int32":
        a = (a < 0.5).to(torch.int32)
    b = torch.empty_like(a)
    key = f"{kw['op']}_{n}"
    out[key] = {}
    for wc, wr in sizes:
        if wc * wr > 1024:
            continue
        ms = st.time(a, b, wc, wr, samples=samples, warmup=1, flush_l2=True)
        out[key][f"{wc}x{wr}"] = round(float(np.median(ms)) * 1e3, 2)
    del a, b
    torch.cuda.empty_cache()
print(json.dumps(out))
