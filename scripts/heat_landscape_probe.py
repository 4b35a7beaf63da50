"""Is heat 16384^2's block-size landscape stable?  Times a handful of sizes
round-robin (flushed single passes, the sweep's measure), several rounds,
and prints per-size medians per round plus the NVML clock/power state.
usage: python scripts/heat_landscape_probe.py [rounds] [samples]"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

from paper_1511_02490_b200 import Stencil

rounds = int(sys.argv[1]) if len(sys.argv) > 1 else 6
samples = int(sys.argv[2]) if len(sys.argv) > 2 else 10
sizes = [(88, 8), (232, 4), (184, 4), (120, 8), (116, 6), (48, 8), (32, 16), (40, 22), (52, 6), (32, 8)]
st = Stencil(op="heat", dtype="float32", border="nearest")
a = torch.rand((16384, 16384), device="cuda")
b = torch.empty_like(a)
try:
    import pynvml as N
    N.nvmlInit()
    h = N.nvmlDeviceGetHandleByIndex(0)
except Exception:
    N = None
res = {f"{c}x{r}": [] for c, r in sizes}
for rd in range(rounds):
    for flush in (True,):
        for c, r in sizes:
            ms = st.time(a, b, c, r, samples=samples, warmup=1, flush_l2=flush)
            res[f"{c}x{r}"].append(float(np.median(ms)))
    if N:
        print("round", rd, "sm", N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM), "MHz, power",
              N.nvmlDeviceGetPowerUsage(h) / 1000, "W", flush=True)
for k, v in res.items():
    print(k, " ".join(f"{x:.4f}" for x in v), " median", f"{np.median(v):.4f}")
# the same with back-to-back (unflushed) passes
for c, r in sizes[:5]:
    ms = st.time(a, b, c, r, samples=samples, warmup=1, flush_l2=False)
    print("noflush", f"{c}x{r}", f"{np.median(ms):.4f}")
