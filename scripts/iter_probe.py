"""Iterated (100 generations, ping-pong) time per generation at several blocks,
against the single-pass sweep's choice: GoL 8192^2 i32 and heat 16384^2 f32."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1511_02490_b200 import Stencil  # noqa: E402

CASES = {"gol": (torch.int32, 8192, "pad", [(36, 28), (32, 32), (60, 8), (48, 16), (128, 8), (24, 32)]),
         "heat": (torch.float32, 16384, "nearest", [(88, 8), (60, 16), (60, 8), (54, 16), (232, 4), (136, 6),
                                                     (104, 8), (32, 16), (48, 8)])}
for op, (dt, n, border, blocks) in CASES.items():
    st = Stencil(op=op, dtype={torch.int32: "int32", torch.float32: "float32"}[dt], border=border)
    a = (torch.rand((n, n), device="cuda") < 0.5).to(dt)
    b = torch.empty_like(a)
    out = {}
    for wc, wr in blocks:
        st.iterate(a, b, 10, wc, wr)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        st.iterate(a, b, 100, wc, wr)
        e1.record()
        torch.cuda.synchronize()
        out[f"{wc}x{wr}"] = round(e0.elapsed_time(e1) / 100 * 1e3, 2)
    print(json.dumps({"workload": op, "us_per_generation": out}), flush=True)
