"""Run `reps` passes of one stencil config (for ncu captures).
usage: python scripts/profile_pass.py op dtype H W wc wr reps [path] [border]"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_1511_02490_b200 import Stencil
op, dtype = sys.argv[1], sys.argv[2]
H, W, wc, wr, reps = map(int, sys.argv[3:8])
path = sys.argv[8] if len(sys.argv) > 8 else "auto"
border = sys.argv[9] if len(sys.argv) > 9 else "pad"
borders = (5, 1, 3, 0) if op == "boxmean" else (1, 1, 1, 1)
st = Stencil(op=op, dtype=dtype, north=borders[0], south=borders[1], east=borders[2],
             west=borders[3], border=border, load_path=path)
tdt = {"int32": torch.int32, "float32": torch.float32, "float64": torch.float64}[dtype]
a = (torch.rand((H, W), device="cuda") < 0.5).to(tdt)
b = torch.empty_like(a)
for _ in range(reps):
    st(a, b, wc, wr)
    a, b = b, a
torch.cuda.synchronize()
print("done", op, dtype, H, W, wc, wr, reps, path)
