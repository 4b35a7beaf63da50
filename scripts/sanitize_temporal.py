"""One small run of each temporally blocked path and of the peer schedule
(one rank: no flag waits, which compute-sanitizer would serialise into a
deadlock), for compute-sanitizer racecheck / memcheck.
usage: python scripts/sanitize_temporal.py {strips|bitplane|fused|peer|streamed}"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

from paper_1511_02490_b200 import Stencil

kind = sys.argv[1]
rng = np.random.default_rng(1)
if kind == "strips":
    st = Stencil(op="heat", dtype="float32", border="nearest", load_path="strips", fused_iterations=5,
                 cells_per_thread=8)
    x = torch.from_numpy(rng.random((77, 301)).astype(np.float32)).cuda()
    st.iterate(x, torch.empty_like(x), 11, 32, 4)
elif kind == "bitplane":
    st = Stencil(op="gol", dtype="int32", load_path="bitplane", fused_iterations=7, cells_per_thread=8)
    x = torch.from_numpy((rng.random((90, 333)) < 0.5).astype(np.int32)).cuda()
    st.iterate(x, torch.empty_like(x), 15, 32, 4)
elif kind == "fused":
    st = Stencil(op="heat", dtype="float32", border="nearest", load_path="tma", fused_iterations=4)
    x = torch.from_numpy(rng.random((70, 128)).astype(np.float32)).cuda()
    st.iterate(x, torch.empty_like(x), 9, 32, 4)
elif kind == "peer":
    from paper_1511_02490_b200.distributed import RowShard, iterate_sharded_peer, local_links, new_control

    st = Stencil(op="heat", dtype="float32", border="nearest")
    sh = RowShard(60, 130, 0, 1, 1, 1)
    a = torch.zeros((sh.buffer_rows, 130), device="cuda")
    a[1:61] = torch.rand((60, 130), device="cuda")
    b = torch.zeros_like(a)
    links = local_links([(a, b, new_control())], [sh])
    iterate_sharded_peer(a, b, sh, 5, st, 32, 4, links[0])
elif kind == "streamed":
    st = Stencil(op="gol", dtype="int32")
    h = [torch.from_numpy((rng.random((64, 96)) < 0.5).astype(np.int32)).pin_memory() for _ in range(4)]
    o = [torch.empty_like(t).pin_memory() for t in h]
    ts = [st.submit_host(h[i], o[i], 3, 32, 4) for i in range(3)]
    st.wait_host(ts[0])
    ts.append(st.submit_host(h[3], o[3], 3, 32, 4))
    for t in ts[1:]:
        st.wait_host(t)
torch.cuda.synchronize()
print("ran", kind)
