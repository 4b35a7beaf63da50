"""Diagnostics: run one stencil configuration in this process and report.
usage: python scripts/probe_paths.py op dtype path wc wr H W [border pad N S E W]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tests"))
import numpy as np
import torch

import oracle_lib as O
from paper_1511_02490_b200 import Stencil

op, dtype, path = sys.argv[1:4]
wc, wr, H, W = map(int, sys.argv[4:8])
border = sys.argv[8] if len(sys.argv) > 8 else "pad"
pad = float(sys.argv[9]) if len(sys.argv) > 9 else 0.0
n, s, e, w = (map(int, sys.argv[10:14]) if len(sys.argv) > 13 else (1, 1, 1, 1))
st = Stencil(op=op, dtype=dtype, north=n, south=s, east=e, west=w, border=border, pad_value=pad,
             load_path=path)
rng = np.random.default_rng(0)
x = (rng.random((H, W)) < 0.5).astype(dtype) if dtype == "int32" else rng.random((H, W)).astype(dtype)
print("probe", st.probe(W, H, wc, wr), flush=True)
a = torch.from_numpy(x).cuda()
b = torch.empty_like(a)
st(a, b, wc, wr)
torch.cuda.synchronize()
want = O.stencil(O.desc_from_stencil(st), x)
print("RESULT", op, dtype, path, wc, wr, "match" if b.cpu().numpy().tobytes() == want.tobytes() else "MISMATCH")
