"""Small runs of the vector work-item kernels (vector.cuh) for compute-sanitizer
memcheck / racecheck / initcheck: every op with a vector form, pad and nearest
borders, ragged grids (edge tiles on all sides), a halo-shard launch, and the
AUTO fallback to the scalar kernel for a misaligned output.
usage: python scripts/sanitize_vector.py"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

from paper_1511_02490_b200 import Stencil

rng = np.random.default_rng(2)
for op, b, dt in [("gol", (1, 1, 1, 1), "int32"), ("heat", (1, 1, 1, 1), "float32"),
                  ("five_point", (1, 1, 1, 1), "float64"), ("sobel", (1, 1, 1, 1), "float32"),
                  ("nms", (1, 1, 1, 1), "int32"), ("boxmean", (5, 1, 3, 0), "float32")]:
    for border in ("pad", "nearest"):
        st = Stencil(op=op, dtype=dt, north=b[0], south=b[1], east=b[2], west=b[3], border=border,
                     pad_value=1.0, load_path="vector")
        x = torch.from_numpy(rng.random((61, 136)).astype(dt)).cuda()
        y = torch.empty_like(x)
        for wc, wr in ((2, 2), (8, 4), (30, 2)):
            st(x, y, wc, wr)
        # halo shard: 3 real rows above and below the 40 computed rows
        st(x[b[0] + 2:], y[b[0] + 2:], 16, 4, rows_above=b[0] + 2, rows_below=b[1] + 2, height=40)
st = Stencil(op="heat", dtype="float32")
x = torch.rand((64, 256), device="cuda")
flat = torch.zeros(64 * 256 + 4, device="cuda")
st(x, flat[1:1 + 64 * 256].view(64, 256), 32, 2)  # AUTO -> scalar TMA (misaligned output)
torch.cuda.synchronize()
print("done")
