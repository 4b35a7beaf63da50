"""A few generations of GoL 8192^2 through (1) one launch per generation and
(2) the fused peer one-pass kernel (one rank, no peers), for ncu captures."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

from paper_1511_02490_b200 import Stencil, fill_host
from paper_1511_02490_b200.distributed import RowShard, iterate_sharded_peer, local_links, new_control

os.environ["SK_PEER_SCHEDULE"] = "fused"
side = 8192
host = np.empty((side, side), dtype=np.int32)
fill_host(host, 2, 2)
st = Stencil(op="gol", dtype="int32")
x = torch.from_numpy(host).cuda()
a, b = x.clone(), torch.empty_like(x)
st.iterate(a, b, 3, 128, 8)
sh = RowShard(side, side, 0, 1, 1, 1)
pa = torch.zeros((sh.buffer_rows, side), dtype=torch.int32, device="cuda")
pa[1:1 + side] = x
pb = torch.zeros_like(pa)
links = local_links([(pa, pb, new_control())], [sh])
iterate_sharded_peer(pa, pb, sh, 3, st, 128, 8, links[0])
torch.cuda.synchronize()
print("done")
