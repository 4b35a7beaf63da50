"""Edge-tile balance of the persistent grid (launch.cu: balanced_grid).  Times
sizes whose tile-column count divides the 148-SM grid (tiles_x = 74 / 37)
next to their neighbours, for heat 16384^2 / 8192^2 and the config-4 box mean,
flushed single passes (the sweep's measure), median of N samples.  Run once
with SK_GRID_BALANCE=0 and once without to compare.
usage: python scripts/grid_balance_probe.py [samples]"""
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

from paper_1511_02490_b200 import Stencil

samples = int(sys.argv[1]) if len(sys.argv) > 1 else 15
cases = [
    (dict(op="heat", dtype="float32", border="nearest"), 16384,
     [(56, 4), (56, 8), (54, 8), (58, 8), (224, 4), (222, 4), (220, 4), (232, 4), (48, 8), (88, 8), (60, 16)]),
    (dict(op="heat", dtype="float32", border="nearest"), 8192,
     [(28, 8), (26, 8), (30, 8), (112, 8), (110, 8), (56, 8), (226, 4)]),
    (dict(op="boxmean", dtype="float32", north=5, south=1, east=3, west=0, border="nearest"), 4096,
     [(16, 8), (32, 4), (24, 16), (28, 8), (8, 8), (64, 4), (96, 4)]),
    (dict(op="gol", dtype="int32"), 8192, [(36, 28), (28, 8), (32, 32)]),
]
out = {"balance": os.environ.get("SK_GRID_BALANCE", "1")}
for kw, n, sizes in cases:
    st = Stencil(**kw)
    a = torch.rand((n, n), device="cuda")
    if kw["dtype"] == "int32":
        a = (a < 0.5).to(torch.int32)
    b = torch.empty_like(a)
    key = f"{kw['op']}_{n}"
    out[key] = {}
    for wc, wr in sizes:
        ms = st.time(a, b, wc, wr, samples=samples, warmup=2, flush_l2=True)
        out[key][f"{wc}x{wr}"] = round(float(np.median(ms)) * 1e3, 2)  # us
    del a, b
    torch.cuda.empty_cache()
print(json.dumps(out))
