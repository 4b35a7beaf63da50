"""Diagnostics: time one pass at every legal size, report failures per size."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_1511_02490_b200 import Stencil
from paper_1511_02490_b200._native import NativeError
st = Stencil(op="gol", dtype="int32")
a = torch.randint(0, 2, (8192, 8192), dtype=torch.int32, device="cuda")
b = torch.empty_like(a)
for wc in range(2, 513, 2):
    for wr in range(2, 1024 // wc + 1, 2):
        try:
            st.time(a, b, wc, wr, samples=1, warmup=0, flush_l2=False)
        except NativeError as e:
            print("FAIL", wc, wr, st.probe(8192, 8192, wc, wr), e, flush=True)
            raise
print("all sizes ok")
