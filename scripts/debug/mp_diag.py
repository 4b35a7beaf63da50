import os, sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
import numpy as np, torch, torch.distributed as dist
import oracle_lib as O
from paper_1511_02490_b200 import Stencil
from paper_1511_02490_b200.distributed import RowShard, cuda_step, iterate_sharded, scatter_rows
dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()
torch.cuda.set_device(0)
n, s, e, w = 3, 2, 1, 0
H, W = 203, 264
rng = np.random.default_rng(5)
full = rng.random((H, W)).astype(np.float32)
st = Stencil(op="boxmean", dtype="float32", north=n, south=s, east=e, west=w, border="nearest")
shard = RowShard(H, W, rank, world, n, s)
from paper_1511_02490_b200.distributed import iterate_sharded_overlapped
if os.environ.get("PRE"):
    sth = Stencil(op="heat", dtype="float32", border="nearest")
    shh = RowShard(H, W, rank, world, 1, 1)
    a2 = scatter_rows(torch.from_numpy(full).cuda(), shh); b2 = torch.zeros_like(a2)
    iterate_sharded_overlapped(a2, b2, shh, 9, sth, 32, 4)
    torch.cuda.synchronize()
    print("pre done", flush=True)
for iters in (1, 2, 3, 9):
    a = scatter_rows(torch.from_numpy(full).cuda(), shard)
    b = torch.zeros_like(a)
    res = iterate_sharded(a, b, shard, iters, cuda_step(st, 32, 4))
    torch.cuda.synchronize()
    want = O.iterate(O.desc_from_stencil(st), full, iters)[shard.r0:shard.r1]
    got = shard.owned(res).cpu().numpy()
    bad = np.argwhere(got != want)
    print(f"rank {rank} iters {iters}: bad {len(bad)} rows {sorted(set(bad[:,0].tolist()))[:8]} halo N {np.abs(a[:n].cpu().numpy()).sum():.3f}", flush=True)
dist.destroy_process_group()
