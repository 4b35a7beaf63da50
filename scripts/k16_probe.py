"""Vector work-items, K = 8 vs K = 16 rows (the K = 16 kernels are 512-thread
bounded: 128 registers): per-pass time over blocks with wr <= 4 (where the
automatic K would allow 16), config-4 box mean 4096^2, GoL 8192^2, heat 16384^2."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1511_02490_b200 import Stencil  # noqa: E402
from paper_1511_02490_b200 import IllegalWorkgroupSize, RefusedParameter  # noqa: E402

WORK = {"boxmean": (dict(op="boxmean", dtype="float32", north=5, south=1, east=3, west=0, border="nearest"), 4096),
        "gol": (dict(op="gol", dtype="int32"), 8192),
        "heat": (dict(op="heat", dtype="float32", border="nearest"), 16384)}
BLOCKS = [(wc, wr) for wc in (8, 16, 24, 32, 48, 60) for wr in (1, 2, 4) if wc * wr >= 16]
for name, (kw, n) in WORK.items():
    a = (torch.rand((n, n), device="cuda") < 0.5).to(torch.int32 if kw["dtype"] == "int32" else torch.float32)
    b = torch.empty_like(a)
    res = {}
    for k in (8, 16):
        st = Stencil(load_path="vector", cells_per_thread=k, **kw)
        best = None
        for wc, wr in BLOCKS:
            try:
                t = sum(st.time(a, b, wc, wr, samples=10, warmup=2)) / 10
            except (IllegalWorkgroupSize, RefusedParameter):
                continue
            if best is None or t < best[0]:
                best = (t, wc, wr)
        res[f"K{k}"] = {"best": f"{best[1]}x{best[2]}", "us": round(best[0] * 1e3, 2)}
    print(json.dumps({"workload": name, **res}), flush=True)
