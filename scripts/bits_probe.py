"""Gcells/s of GoL 8192^2 x 100 generations on the bit-plane path over
(TB, wc, wr, K); CUDA events, inputs larger than L2.
usage: python scripts/bits_probe.py [side] [iters] [dtype]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

from paper_1511_02490_b200 import IllegalWorkgroupSize, NativeError, RefusedParameter, Stencil, fill_host
import numpy as np

side = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 100
dtype = sys.argv[3] if len(sys.argv) > 3 else "int32"
tdt = {"int32": torch.int32, "float32": torch.float32, "float64": torch.float64}[dtype]
host = np.empty((side, side), dtype=np.int32)
fill_host(host, 2, 2)
a0 = torch.from_numpy(host).to(tdt).cuda()
ref = Stencil(op="gol", dtype=dtype)
want = ref.iterate(a0.clone(), torch.empty_like(a0), iters, 32, 8).clone()
rows = []
import itertools
cfgs = [(tb, wc, wr, k) for tb in (4, 6, 8, 10, 13, 17, 20, 25, 34)
        for (wc, wr) in [(32, 1), (32, 2), (32, 4), (32, 8), (32, 16), (32, 24), (64, 8), (32, 12), (32, 6)]
        for k in (16, 32)]
for tb, wc, wr, k in cfgs:
    if True:
        if True:
            st = Stencil(op="gol", dtype=dtype, fused_iterations=tb, load_path="bitplane",
                         cells_per_thread=k)
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
            g = side * side * iters / (ms / 1e3) / 1e9
            rows.append((g, tb, wc, wr, k, ms, ok))
rows.sort(reverse=True)
print("bad:", [r for r in rows if not r[6]][:5])
for g, tb, wc, wr, k, ms, ok in rows[:30]:
    print(f"{dtype} {side}^2 x{iters}: TB={tb:3d} {wc}x{wr} K={k}: {g:9.1f} Gcells/s ({ms:.3f} ms) ok={ok}")
for tb in sorted({c[0] for c in cfgs}):
    best = max((r for r in rows if r[1] == tb), default=None)
    print(f"best TB={tb}: {best}")
