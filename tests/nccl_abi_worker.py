"""Worker for tests/test_nccl_halo.py (run under torchrun, NCCL backend, one
GPU per rank): row-sharded heat / GoL / boxmean through the C-ABI NCCL
schedule (iterate_sharded_nccl -> sk_stencil_iterate_nccl with torch's
ncclComm_t), gathered on rank 0 and compared bit for bit with the CPU
oracle."""
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import numpy as np
import torch
import torch.distributed as dist

import oracle_lib as O
from paper_1511_02490_b200 import Stencil
from paper_1511_02490_b200.distributed import RowShard, iterate_sharded_nccl, scatter_rows


def main():
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, world = dist.get_rank(), dist.get_world_size()
    ok = True
    for op, dtype, border, borders in [("heat", "float32", "nearest", (1, 1, 1, 1)),
                                       ("gol", "int32", "pad", (1, 1, 1, 1)),
                                       ("boxmean", "float32", "nearest", (5, 1, 3, 0))]:
        n, s, e, w = borders
        H, W, iters = 301, 520, 7
        rng = np.random.default_rng(9)
        full = (rng.random((H, W)) < 0.4).astype(np.int32) if dtype == "int32" else \
            rng.random((H, W)).astype(dtype)
        st = Stencil(op=op, dtype=dtype, north=n, south=s, east=e, west=w, border=border)
        shard = RowShard(H, W, rank, world, n, s)
        a = scatter_rows(torch.from_numpy(full).cuda(), shard)
        b = torch.zeros_like(a)
        dist.barrier()  # the communicator exists before the library uses it
        res = iterate_sharded_nccl(a, b, shard, iters, st, 32, 4)
        torch.cuda.synchronize()
        # shards differ by a row: gather padded blocks, then trim
        rows = [RowShard(H, W, r, world, n, s).rows for r in range(world)]
        mine = torch.zeros((max(rows), W), dtype=res.dtype, device="cuda")
        mine[:shard.rows] = shard.owned(res)
        parts = [torch.empty_like(mine) for _ in range(world)]
        dist.all_gather(parts, mine)
        if rank == 0:
            got = torch.cat([p[:r] for p, r in zip(parts, rows)]).cpu().numpy()
            want = O.iterate(O.desc_from_stencil(st), full, iters)
            same = got.tobytes() == want.tobytes()
            print(f"{op}: {'ok' if same else 'MISMATCH'} (world {world})", flush=True)
            ok = ok and same
    dist.barrier()
    if rank == 0 and ok:
        print("ALL_OK", flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
