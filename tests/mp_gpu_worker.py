"""Worker for tests/test_multirank_gpu.py (run under torchrun): row-sharded
GoL / heat on the CUDA executor with halo exchange, gathered on rank 0 and
compared bit-for-bit with the CPU oracle.  Uses gloo (host-staged halos) so
2 ranks can share the single GPU of a gpurun box; NCCL is the production
transport and uses the same exchange code."""
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
from paper_1511_02490_b200.distributed import (RowShard, cuda_step, iterate_sharded,
                                               iterate_sharded_overlapped, scatter_rows)


def main():
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(0)
    ok = True
    for op, dtype, border, borders in [("gol", "int32", "pad", (1, 1, 1, 1)),
                                       ("heat", "float32", "nearest", (1, 1, 1, 1)),
                                       ("boxmean", "float32", "nearest", (3, 2, 1, 0))]:
        n, s, e, w = borders
        H, W, iters = 203, 264, 9
        rng = np.random.default_rng(5)
        full = (rng.random((H, W)) < 0.4).astype(np.int32) if dtype == "int32" else \
            rng.random((H, W)).astype(dtype)
        st = Stencil(op=op, dtype=dtype, north=n, south=s, east=e, west=w, border=border)
        shard = RowShard(H, W, rank, world, n, s)
        a = scatter_rows(torch.from_numpy(full).cuda(), shard)
        b = torch.zeros_like(a)
        res = iterate_sharded(a, b, shard, iters, cuda_step(st, 32, 4))
        torch.cuda.synchronize()
        part = shard.owned(res).cpu()
        a2 = scatter_rows(torch.from_numpy(full).cuda(), shard)
        b2 = torch.zeros_like(a2)
        res2 = iterate_sharded_overlapped(a2, b2, shard, iters, st, 32, 4)
        torch.cuda.synchronize()
        same_overlap = bool(torch.equal(shard.owned(res2), shard.owned(res)))
        parts = [None] * world
        dist.all_gather_object(parts, (shard.r0, part.numpy(), same_overlap))
        if rank == 0:
            got = np.concatenate([p[1] for p in sorted(parts, key=lambda t: t[0])])
            want = O.iterate(O.desc_from_stencil(st), full, iters)
            same = got.tobytes() == want.tobytes() and all(p[2] for p in parts)
            print(f"{op}: {'match' if same else 'MISMATCH'} (overlapped: {[p[2] for p in parts]})",
                  flush=True)
            if not same:
                bad = np.argwhere(got != want)
                print(f"  {len(bad)} cells differ; rows {sorted(set(bad[:, 0].tolist()))[:12]}",
                      flush=True)
            ok = ok and same
    if rank == 0:
        print("ALL_OK" if ok else "FAILED", flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
