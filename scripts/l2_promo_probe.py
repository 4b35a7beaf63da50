"""TMA L2 fill granularity (launch.cu: l2_promotion, SK_L2_PROMO) vs tile
shape: heat 16384^2 vector sizes whose DRAM reads exceed the algorithmic bytes
(48x8: 1.25 GB vs 1.07), their neighbours, the scalar best, GoL and the
config-4 box mean at their oracle blocks.  Flushed single passes, median (us).
usage: SK_L2_PROMO=<0|64|128|256> python scripts/l2_promo_probe.py [samples]"""
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
     [(48, 8), (52, 8), (54, 8), (40, 8), (32, 16), (60, 16), (32, 4), (88, 8), (232, 4), (160, 6)]),
    (dict(op="gol", dtype="int32"), 8192, [(36, 28), (32, 28), (32, 32), (48, 16), (128, 8)]),
    (dict(op="boxmean", dtype="float32", north=5, south=1, east=3, west=0, border="nearest"), 4096,
     [(16, 8), (32, 4)]),
]
out = {"l2_promo": os.environ.get("SK_L2_PROMO", "256")}
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
        out[key][f"{wc}x{wr}"] = round(float(np.median(ms)) * 1e3, 2)
    del a, b
    torch.cuda.empty_cache()
print(json.dumps(out))
