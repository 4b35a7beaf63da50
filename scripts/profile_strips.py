"""Run `reps` iterate() calls of heat on the register-strip path (for ncu
captures).  usage: python scripts/profile_strips.py side tb k wc wr reps"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_1511_02490_b200 import Stencil
side, tb, k, wc, wr, reps = map(int, sys.argv[1:7])
st = Stencil(op="heat", dtype="float32", border="nearest", load_path="strips", fused_iterations=tb,
             cells_per_thread=k)
a = torch.rand((side, side), device="cuda")
b = torch.empty_like(a)
for _ in range(reps):
    st.iterate(a, b, 3 * tb, wc, wr)
torch.cuda.synchronize()
print("done", side, tb, k, wc, wr, reps)
