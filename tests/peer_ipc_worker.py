"""Two-process check of the IPC-mapped peer exchange (run by
tests/test_peer_halo.py::test_peer_exchange_two_processes_ipc): the ranks
share cuda:0, rendezvous over gloo, export / import their buffers with CUDA
IPC handles and run sk_stencil_iterate_peer; rank 0 gathers the grid and
compares it with the CPU oracle bit for bit."""
from __future__ import annotations

import os
import sys

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def worker(rank: int, world: int, result) -> None:
    import oracle_lib as O
    from paper_1511_02490_b200 import Stencil
    from paper_1511_02490_b200.distributed import RowShard, connect_peers, iterate_sharded_peer, new_control

    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    H, W, iters = 96, 130, 6
    rng = np.random.default_rng(5)
    x = (2 * rng.random((H, W)) - 1).astype(np.float32)
    st = Stencil(op="heat", dtype="float32", border="nearest")
    sh = RowShard(H, W, rank, world, 1, 1)
    a = torch.zeros((sh.buffer_rows, W), dtype=torch.float32, device="cuda")
    a[1:1 + sh.rows] = torch.from_numpy(x[sh.r0:sh.r1]).cuda()
    b = torch.zeros_like(a)
    links = connect_peers(a, b, new_control(), sh)
    res = iterate_sharded_peer(a, b, sh, iters, st, 32, 8, links)
    torch.cuda.synchronize()
    dist.barrier()
    parts = [None] * world
    dist.all_gather_object(parts, sh.owned(res).cpu().numpy())
    dist.barrier()
    links.close()
    if rank == 0:
        got = np.concatenate(parts)
        want = O.iterate(O.desc_from_stencil(st), x, iters)
        result.value = int(got.tobytes() == want.tobytes())
    dist.destroy_process_group()


def main() -> int:
    ctx = mp.get_context("spawn")
    result = ctx.Value("i", -1)
    procs = [ctx.Process(target=worker, args=(r, 2, result)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(180)
        if p.is_alive():
            p.kill()
            print("peer-ipc: timeout")
            return 1
    if any(p.exitcode for p in procs) or result.value != 1:
        print(f"peer-ipc: failed (exit codes {[p.exitcode for p in procs]}, match={result.value})")
        return 1
    print("peer-ipc: ok")
    return 0


if __name__ == "__main__":
    sys.exit(main())
