"""Upper bound on what edge tiles cost: the same kernel and block with the
zero-pad border (TMA zero fill, no fix-up, no barriers) against the nearest
border (fix-ups between two block barriers).  Flushed passes, median (us).
usage: python scripts/edge_cost_probe.py [samples]"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

from paper_1511_02490_b200 import Stencil

samples = int(sys.argv[1]) if len(sys.argv) > 1 else 21
out = {}
for op, n, kw, sizes in [("boxmean", 4096, dict(north=5, south=1, east=3, west=0), [(16, 8), (32, 4), (8, 8)]),
                         ("heat", 16384, {}, [(54, 8), (88, 8), (48, 8)]),
                         ("heat", 4096, {}, [(54, 8), (88, 8)])]:
    a = torch.rand((n, n), device="cuda")
    b = torch.empty_like(a)
    for border in ("pad", "nearest"):
        st = Stencil(op=op, dtype="float32", border=border, **kw)
        for wc, wr in sizes:
            ms = st.time(a, b, wc, wr, samples=samples, warmup=2, flush_l2=True)
            out[f"{op}_{n}_{wc}x{wr}_{border}"] = round(float(np.median(ms)) * 1e3, 2)
print(json.dumps(out))
