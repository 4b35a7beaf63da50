"""Run `reps` iterate() calls of bit-plane GoL (for ncu captures): with
iterations = 3*TB each call is T->bits, bits->bits, bits->T launches.
usage: python scripts/profile_bits.py side tb wc wr k reps"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_1511_02490_b200 import Stencil
side, tb, wc, wr, k, reps = map(int, sys.argv[1:7])
st = Stencil(op="gol", dtype="int32", fused_iterations=tb, load_path="bitplane", cells_per_thread=k)
a = (torch.rand((side, side), device="cuda") < 0.5).to(torch.int32)
b = torch.empty_like(a)
for _ in range(reps):
    st.iterate(a, b, 3 * tb, wc, wr)
torch.cuda.synchronize()
print("done", side, tb, wc, wr, k, reps)
