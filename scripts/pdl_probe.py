"""Per-generation time of the one-pass loop with and without programmatic
dependent launch (run twice: SK_PDL=0 and default), GoL 8192^2 at 36x28 and
32x32, heat 16384^2 at 116x6, box mean 4096^2 at 16x8 - through
Stencil.iterate (graph replay) and through per-generation launches."""
import json
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1511_02490_b200 import Stencil  # noqa: E402

CASES = [("gol", torch.int32, 8192, dict(), [(36, 28), (32, 32)]),
         ("heat", torch.float32, 16384, dict(border="nearest"), [(116, 6)]),
         ("boxmean", torch.float32, 4096, dict(north=5, south=1, east=3, west=0, border="nearest"), [(16, 8)])]
out = {"pdl": os.environ.get("SK_PDL", "1")}
for op, dt, n, kw, blocks in CASES:
    st = Stencil(op=op, dtype="int32" if dt == torch.int32 else "float32", **kw)
    a = (torch.rand((n, n), device="cuda") < 0.5).to(dt)
    b = torch.empty_like(a)
    for wc, wr in blocks:
        for mode in ("iterate", "launches"):
            def run(k):
                if mode == "iterate":
                    st.iterate(a, b, k, wc, wr)
                else:
                    x, y = a, b
                    for _ in range(k):
                        st(x, y, wc, wr)
                        x, y = y, x
            for _ in range(3):
                run(20)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            run(200)
            e1.record()
            torch.cuda.synchronize()
            out[f"{op}_{wc}x{wr}_{mode}"] = round(e0.elapsed_time(e1) / 200 * 1e3, 2)
print(json.dumps(out), flush=True)
