"""Gcells/s of heat / five_point on the register-strip path over (TB, K, wc,
wr) on a side^2 grid, `iters` generations, CUDA events, inputs larger than L2;
each configuration is checked bit-exact against the one-pass executor.
usage: python scripts/strips_probe.py [op] [dtype] [side] [iters] [tb,tb,...]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

from paper_1511_02490_b200 import IllegalWorkgroupSize, NativeError, RefusedParameter, Stencil, fill_host

op = sys.argv[1] if len(sys.argv) > 1 else "heat"
dtype = sys.argv[2] if len(sys.argv) > 2 else "float32"
side = int(sys.argv[3]) if len(sys.argv) > 3 else 16384
iters = int(sys.argv[4]) if len(sys.argv) > 4 else 100
tdt = {"int32": torch.int32, "float32": torch.float32, "float64": torch.float64}[dtype]
host = np.empty((side, side), dtype=dtype)
fill_host(host, 1 if dtype != "int32" else 2, 3)
a0 = torch.from_numpy(host).cuda()
one = Stencil(op=op, dtype=dtype, border="nearest")
want = one.iterate(a0.clone(), torch.empty_like(a0), iters, 64, 8).clone()
rows = []
TBS = [int(t) for t in sys.argv[5].split(",")] if len(sys.argv) > 5 else [4, 6, 8, 10, 12, 16]
for tb in TBS:
    for k in (4, 8, 16):
        for wc, wr in [(32, 4), (32, 6), (32, 8), (32, 12), (32, 16), (32, 24), (64, 8), (32, 32)]:
            st = Stencil(op=op, dtype=dtype, border="nearest", load_path="strips",
                         fused_iterations=tb, cells_per_thread=k)
            a, b = a0.clone(), torch.empty_like(a0)
            try:
                res = st.iterate(a, b, iters, wc, wr)
                torch.cuda.synchronize()
                ok = torch.equal(res, want)
                ts = []
                for _ in range(3):
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    st.iterate(a, b, iters, wc, wr)
                    e1.record()
                    torch.cuda.synchronize()
                    ts.append(e0.elapsed_time(e1))
            except (IllegalWorkgroupSize, RefusedParameter, NativeError):
                continue
            ms = min(ts)
            rows.append((side * side * iters / (ms / 1e3) / 1e9, tb, k, wc, wr, ms, ok))
rows.sort(reverse=True)
print("bad:", [r for r in rows if not r[6]][:5])
for g, tb, k, wc, wr, ms, ok in rows[:25]:
    print(f"{op} {dtype} {side}^2 x{iters}: TB={tb:2d} K={k:2d} {wc}x{wr}: {g:8.1f} Gcells/s ({ms:.3f} ms) ok={ok}")
for tb in sorted({r[1] for r in rows}):
    print(f"best TB={tb}: {max(r for r in rows if r[1] == tb)}")
