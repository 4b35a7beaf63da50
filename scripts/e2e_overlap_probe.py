"""Where the e2e path (streamed host jobs) loses against the device-only step:
GoL 8192^2 x 100 at 32x28.  Times (1) one job's 100 generations on device
buffers, (2) the same while a 268 MB H2D and a 268 MB D2H run on side streams
(copy-engine traffic sharing HBM), (3) the copies alone, (4) the streamed
host API with 2 and 3 jobs in flight.
usage: python scripts/e2e_overlap_probe.py"""
import json
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1511_02490_b200 import Stencil  # noqa: E402

st = Stencil(op="gol", dtype="int32")
W = H = 8192
WC, WR, G = 32, 28, 100
host = (torch.rand((H, W)) < 0.5).to(torch.int32)
h_in = [host.clone().pin_memory() for _ in range(3)]
h_out = [torch.empty_like(host).pin_memory() for _ in range(3)]
a = host.cuda()
b = torch.empty_like(a)
c = torch.empty_like(a)
s_h2d, s_d2h = torch.cuda.Stream(), torch.cuda.Stream()
out = {}


def timed(fn, reps=5):
    best = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best.append(time.perf_counter() - t0)
    return sorted(best)[len(best) // 2] * 1e3


st.iterate(a, b, G, WC, WR)
out["compute_ms"] = round(timed(lambda: st.iterate(a, b, G, WC, WR)), 3)


def with_copies():
    with torch.cuda.stream(s_h2d):
        c.copy_(h_in[0], non_blocking=True)
    with torch.cuda.stream(s_d2h):
        h_out[0].copy_(b, non_blocking=True)
    st.iterate(a, b, G, WC, WR)


out["compute_with_copies_ms"] = round(timed(with_copies), 3)
out["h2d_ms"] = round(timed(lambda: c.copy_(h_in[0], non_blocking=True)), 3)
out["d2h_ms"] = round(timed(lambda: h_out[0].copy_(b, non_blocking=True)), 3)


def both_copies():
    with torch.cuda.stream(s_h2d):
        c.copy_(h_in[0], non_blocking=True)
    with torch.cuda.stream(s_d2h):
        h_out[0].copy_(b, non_blocking=True)


out["h2d_and_d2h_ms"] = round(timed(both_copies), 3)
for depth in (2, 3):
    for j in range(3):
        st.wait_host(st.submit_host(h_in[j], h_out[j], G, WC, WR))
    k = 48
    tickets = []
    t0 = time.perf_counter()
    for j in range(k):
        if len(tickets) >= depth:
            st.wait_host(tickets.pop(0))
        tickets.append(st.submit_host(h_in[j % 3], h_out[j % 3], G, WC, WR))
    for t in tickets:
        st.wait_host(t)
    dt = time.perf_counter() - t0
    out[f"streamed_depth{depth}_ms_per_job"] = round(dt / k * 1e3, 3)
    out[f"streamed_depth{depth}_gcells"] = round(W * H * G * k / dt / 1e9, 1)
out["device_only_gcells"] = round(W * H * G / out["compute_ms"] * 1e-6, 1)
print(json.dumps(out), flush=True)
