"""Per-generation cost of the peer schedule's split (boundary strips + interior
launch) against one launch per generation, on one GPU with one rank (no
peers: the strips still run, the flags are not waited on).
usage: python scripts/peer_overhead_probe.py [side] [iters] [wc] [wr]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

from paper_1511_02490_b200 import Stencil, fill_host
from paper_1511_02490_b200.distributed import RowShard, iterate_sharded_peer, local_links, new_control

side = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 100
wc = int(sys.argv[3]) if len(sys.argv) > 3 else 128
wr = int(sys.argv[4]) if len(sys.argv) > 4 else 8
host = np.empty((side, side), dtype=np.int32)
fill_host(host, 2, 2)
st = Stencil(op="gol", dtype="int32")
x = torch.from_numpy(host).cuda()


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


a, b = x.clone(), torch.empty_like(x)
one = timed(lambda: st.iterate(a, b, iters, wc, wr))
sh = RowShard(side, side, 0, 1, 1, 1)
pa = torch.zeros((sh.buffer_rows, side), dtype=torch.int32, device="cuda")
pa[1:1 + side] = x
pb = torch.zeros_like(pa)
links = local_links([(pa, pb, new_control())], [sh])
peer = timed(lambda: iterate_sharded_peer(pa, pb, sh, iters, st, wc, wr, links[0]))
print(f"one launch per generation: {one / iters * 1e3:.2f} us/gen")
print(f"peer schedule (strips + interior): {peer / iters * 1e3:.2f} us/gen "
      f"(+{(peer - one) / iters * 1e3:.2f} us, {100 * (peer / one - 1):.1f} %)")
