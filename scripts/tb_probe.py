"""Measure iterated throughput (Gcells/s) with and without temporal blocking.
usage: python scripts/tb_probe.py [op] [dtype] [side] [iters]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

from paper_1511_02490_b200 import IllegalWorkgroupSize, NativeError, RefusedParameter, Stencil

op = sys.argv[1] if len(sys.argv) > 1 else "gol"
dtype = sys.argv[2] if len(sys.argv) > 2 else "int32"
side = int(sys.argv[3]) if len(sys.argv) > 3 else 8192
iters = int(sys.argv[4]) if len(sys.argv) > 4 else 100
border = "pad" if op == "gol" else "nearest"
tdt = {"int32": torch.int32, "float32": torch.float32, "float64": torch.float64}[dtype]
a0 = (torch.rand((side, side), device="cuda") < 0.5).to(tdt)
rows = []
for tb in (1, 2, 4):
    for k in (0, 4, 8):
        for wc, wr in [(32, 8), (64, 4), (96, 6), (128, 4), (64, 8), (32, 16), (128, 2), (256, 2), (64, 16), (32, 4)]:
            st = Stencil(op=op, dtype=dtype, border=border, fused_iterations=tb, cells_per_thread=k)
            a, b = a0.clone(), torch.empty_like(a0)
            try:
                st.iterate(a, b, 4, wc, wr)
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                st.iterate(a, b, iters, wc, wr)
                e1.record()
                torch.cuda.synchronize()
            except (IllegalWorkgroupSize, RefusedParameter, NativeError):
                continue
            ms = e0.elapsed_time(e1)
            g = side * side * iters / (ms / 1e3) / 1e9
            rows.append((g, tb, k, wc, wr, ms))
rows.sort(reverse=True)
for g, tb, k, wc, wr, ms in rows[:15]:
    print(f"{op} {dtype} {side}^2 x{iters}: TB={tb} K={k} {wc}x{wr}: {g:8.1f} Gcells/s ({ms:.2f} ms)")
for tb in (1, 2, 4):
    best = max((r for r in rows if r[1] == tb), default=None)
    print(f"best TB={tb}: {best}")
