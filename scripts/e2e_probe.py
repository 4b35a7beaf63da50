"""End-to-end throughput of the streamed host API (sk_stencil_submit_host /
sk_stencil_wait_host, three jobs in flight) for GoL 8192^2 x 100 from pinned
buffers, against the number of jobs in the measurement (pipeline fill and
drain amortisation), plus the copy-only and compute-only times of one job."""
import json
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1511_02490_b200 import Stencil  # noqa: E402

st = Stencil(op="gol", dtype="int32")
W = H = 8192
host = (torch.rand((H, W)) < 0.5).to(torch.int32)
h_in = [host.clone().pin_memory() for _ in range(3)]
h_out = [torch.empty_like(host).pin_memory() for _ in range(3)]
for j in range(3):
    st.wait_host(st.submit_host(h_in[j], h_out[j], 100, 36, 28))
d = torch.empty_like(host, device="cuda")
torch.cuda.synchronize()
t0 = time.perf_counter(); d.copy_(h_in[0], non_blocking=True); torch.cuda.synchronize(); h2d = time.perf_counter() - t0
t0 = time.perf_counter(); h_out[0].copy_(d, non_blocking=True); torch.cuda.synchronize(); d2h = time.perf_counter() - t0
out = {"h2d_ms": round(h2d * 1e3, 2), "d2h_ms": round(d2h * 1e3, 2)}
for k in (6, 12, 24, 48, 96):
    tickets = []
    t0 = time.perf_counter()
    for j in range(k):
        if len(tickets) >= 3:
            st.wait_host(tickets.pop(0))
        tickets.append(st.submit_host(h_in[j % 3], h_out[j % 3], 100, 36, 28))
    for t in tickets:
        st.wait_host(t)
    dt = time.perf_counter() - t0
    out[f"jobs_{k}"] = round(W * H * 100 * k / dt / 1e9, 1)
print(json.dumps(out), flush=True)
