"""Per-generation time of P single-process ranks (one GPU, one stream each)
running the peer schedule over a shared grid, against one launch per
generation over the undivided grid - a one-GPU proxy for the multi-GPU
overhead of each schedule (the ranks' kernels share the GPU, so the total
work equals the undivided pass).  SK_PEER_SCHEDULE=strips forces the
strips + interior schedule; default is the fused one-pass kernel.
usage: python scripts/peer_ranks_probe.py [ranks] [side] [iters] [wc] [wr]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

from paper_1511_02490_b200 import Stencil, fill_host
from paper_1511_02490_b200.distributed import RowShard, iterate_sharded_peer, local_links, new_control

P = int(sys.argv[1]) if len(sys.argv) > 1 else 2
side = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 100
wc = int(sys.argv[4]) if len(sys.argv) > 4 else 128
wr = int(sys.argv[5]) if len(sys.argv) > 5 else 8
host = np.empty((side, side), dtype=np.int32)
fill_host(host, 2, 2)
st = Stencil(op="gol", dtype="int32")
x = torch.from_numpy(host).cuda()
a, b = x.clone(), torch.empty_like(x)

shards = [RowShard(side, side, p, P, 1, 1) for p in range(P)]
bufs, streams = [], []
for sh in shards:
    pa = torch.zeros((sh.buffer_rows, side), dtype=torch.int32, device="cuda")
    pa[1:1 + sh.rows] = x[sh.r0:sh.r1]
    bufs.append((pa, torch.zeros_like(pa), new_control()))
    streams.append(torch.cuda.Stream())
links = local_links(bufs, shards)
cur = [(p_a, p_b) for p_a, p_b, _ in bufs]


def ranks_step():
    for p, sh in enumerate(shards):
        ra, rb = cur[p]
        res = iterate_sharded_peer(ra, rb, sh, iters, st, wc, wr, links[p], stream=streams[p])
        cur[p] = (res, rb if res is ra else ra)


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    for s in streams:
        torch.cuda.current_stream().wait_stream(s)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


one = timed(lambda: st.iterate(a, b, iters, wc, wr))
many = timed(ranks_step)
want = st.iterate(x.clone(), torch.empty_like(x), iters * 6, wc, wr)
got = torch.cat([sh.owned(cur[p][0]) for p, sh in enumerate(shards)])
print(f"undivided, one launch per generation: {one / iters * 1e3:.2f} us/gen")
print(f"{P} ranks, peer schedule: {many / iters * 1e3:.2f} us/gen ({100 * (many / one - 1):+.1f} %), "
      f"bit-exact={bool(torch.equal(got, want))}")
