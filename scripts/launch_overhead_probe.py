"""Per-generation time of sk_stencil_iterate on small grids (where launches,
not HBM, bound the loop): GoL 64^2 / 256^2 / 1024^2 / 2048^2 i32, heat 1024^2."""
import json
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1511_02490_b200 import Stencil  # noqa: E402

for op, dt, n in [("gol", torch.int32, 64), ("gol", torch.int32, 256), ("gol", torch.int32, 1024),
                  ("gol", torch.int32, 2048), ("heat", torch.float32, 1024)]:
    st = Stencil(op=op, dtype="int32" if dt == torch.int32 else "float32")
    a = (torch.rand((n, n), device="cuda") < 0.5).to(dt)
    b = torch.empty_like(a)
    for _ in range(2):  # first call: direct (+ graph capture when enabled)
        st.iterate(a, b, 1000, 32, 8)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    st.iterate(a, b, 1000, 32, 8)
    e1.record()
    host = (time.perf_counter() - t0) / 1000 * 1e6
    torch.cuda.synchronize()
    print(json.dumps({"op": op, "n": n, "gpu_us_per_gen": round(e0.elapsed_time(e1), 3),
                      "host_us_per_launch_call": round(host, 2)}), flush=True)
