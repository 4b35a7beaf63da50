"""Repeat one stencil configuration many times and count runs whose output
differs from the CPU oracle (hunts intermittent races).
usage: python scripts/stress_race.py op dtype H W wc wr reps [border] [k] [path] [stages_env]"""
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import numpy as np
import torch

import oracle_lib as O
from paper_1511_02490_b200 import Stencil, fill_host

op, dtype = sys.argv[1], sys.argv[2]
H, W, wc, wr, reps = map(int, sys.argv[3:8])
border = sys.argv[8] if len(sys.argv) > 8 else "nearest"
k = int(sys.argv[9]) if len(sys.argv) > 9 else 0
path = sys.argv[10] if len(sys.argv) > 10 else "auto"
st = Stencil(op=op, dtype=dtype, border=border, cells_per_thread=k, load_path=path)
x = np.empty((H, W), dtype)
fill_host(x, 2 if op == "gol" else (3 if dtype == "int32" else 0), 1)
want = torch.from_numpy(O.stencil(O.desc_from_stencil(st), x, threads=os.cpu_count() or 8)).cuda()
a = torch.from_numpy(x).cuda()
outs = [torch.empty_like(a) for _ in range(8)]
bad = 0
where = []
for i in range(reps):
    b = outs[i % 8]
    b.fill_(-7)
    st(a, b, wc, wr)
    if i % 8 == 7 or i == reps - 1:
        for j, bb in enumerate(outs[: (i % 8) + 1]):
            if not torch.equal(bb, want):
                bad += 1
                idx = (bb != want).nonzero()[:4].tolist()
                where.append(idx)
print(f"RESULT {op} {dtype} {H}x{W} {wc}x{wr} k={k} {path} {border}: {bad}/{reps} bad; first {where[:3]}",
      st.probe(W, H, wc, wr), flush=True)
