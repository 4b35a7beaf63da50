"""One-pass GoL 8192^2: mean pass time (30 samples, L2 flushed) for K = 8 and
K = 16 cells per work-item over a set of block shapes.
usage: python scripts/k_probe.py"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

from paper_1511_02490_b200 import IllegalWorkgroupSize, RefusedParameter, Stencil

a = (torch.rand((8192, 8192), device="cuda") < 0.5).to(torch.int32)
b = torch.empty_like(a)
want = Stencil(op="gol", dtype="int32", cells_per_thread=8).iterate(a.clone(), torch.empty_like(a), 3, 128, 8).clone()
rows = []
for wc, wr in [(128, 8), (144, 4), (128, 4), (256, 4), (96, 4), (64, 4), (128, 2), (256, 2), (192, 4), (160, 4),
               (64, 8), (96, 6), (512, 2), (32, 4), (320, 2), (384, 2)]:
    for k in (8, 16):
        st = Stencil(op="gol", dtype="int32", cells_per_thread=k)
        try:
            ms = st.time(a, b, wc, wr, samples=30, warmup=3, flush_l2=True)
            ok = torch.equal(st.iterate(a.clone(), torch.empty_like(a), 3, wc, wr), want)
        except (IllegalWorkgroupSize, RefusedParameter):
            continue
        m = sum(ms) / len(ms)
        rows.append((m, wc, wr, k, ok))
rows.sort()
for m, wc, wr, k, ok in rows[:16]:
    print(f"gol 8192^2 {wc}x{wr} K={k}: {m*1e3:.1f} us, {8192*8192/(m/1e3)/1e9:.1f} Gcells/s, "
          f"{100*8192*8192*8/(m/1e3)/1e9/6533.2:.1f}% HBM, exact={ok}")
