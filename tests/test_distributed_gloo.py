"""Multi-process (gloo, CPU) test of the row-block decomposition with halo
exchange (paper_1511_02490_b200/distributed.py): P ranks iterating their
shards with per-iteration halo exchange must reproduce the undivided run
bit-for-bit.  The per-shard compute here is the CPU oracle (the checker); on
B200 the same exchange drives the CUDA executor over NCCL."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle_lib as O
from paper_1511_02490_b200.distributed import (RowShard, iterate_sharded,
                                               iterate_sharded_overlapped, scatter_rows)

CASES = {
    "gol": dict(op="gol", dtype="int32", n=1, s=1, e=1, w=1, border="pad", pad=0.0),
    "heat": dict(op="heat", dtype="float32", n=1, s=1, e=1, w=1, border="nearest", pad=0.0),
    "asym": dict(op="boxmean", dtype="float64", n=3, s=2, e=1, w=0, border="nearest", pad=0.0),
    "padded": dict(op="boxmean", dtype="float32", n=2, s=3, e=2, w=2, border="pad", pad=0.5),
}
H, W, ITERS = 61, 45, 7


def make_grid(c):
    rng = np.random.default_rng(17)
    if c["dtype"] == "int32":
        return (rng.random((H, W)) < 0.45).astype(np.int32)
    return rng.random((H, W)).astype(c["dtype"])


def oracle_desc(c):
    return O.desc_from(c["op"], c["dtype"], c["n"], c["s"], c["e"], c["w"], c["border"], c["pad"])


def oracle_step(desc):
    def step(src, dst, shard):
        lo = shard.north - shard.rows_above
        hi = shard.north + shard.rows + shard.rows_below
        window = src[lo:hi].numpy()
        out = O.stencil(desc, window, rows_above=shard.rows_above, rows_below=shard.rows_below,
                        threads=1)
        dst[shard.north:shard.north + shard.rows] = torch.from_numpy(out)
    return step


class OracleStencil:
    """The executor's call signature (Stencil.__call__) over the CPU oracle,
    so the overlapped schedule's strip/exchange logic runs on host tensors."""

    def __init__(self, desc):
        self.desc = desc

    def __call__(self, src, dst, wc, wr, rows_above=0, rows_below=0, height=None):
        base = src.storage_offset()
        full = src.as_strided((src.shape[0] + rows_above, src.shape[1]), src.stride(),
                              base - rows_above * src.stride(0))
        win = full[:rows_above + height + rows_below].numpy()
        out = O.stencil(self.desc, win, rows_above=rows_above, rows_below=rows_below, threads=1)
        dst[:height] = torch.from_numpy(out)


def worker(rank, world, port, case, q, overlapped=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        c = CASES[case]
        full = torch.from_numpy(make_grid(c))
        shard = RowShard(H, W, rank, world, c["n"], c["s"])
        a = scatter_rows(full, shard)
        b = torch.zeros_like(a)
        if overlapped:
            res = iterate_sharded_overlapped(a, b, shard, ITERS, OracleStencil(oracle_desc(c)), 0, 0)
        else:
            res = iterate_sharded(a, b, shard, ITERS, oracle_step(oracle_desc(c)))
        q.put((rank, shard.r0, shard.owned(res).clone().numpy()))
    finally:
        dist.destroy_process_group()


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("overlapped", [False, True], ids=["serial", "overlapped"])
@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("case", sorted(CASES))
def test_sharded_iteration_matches_single(world, case, overlapped):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, world, port, case, q, overlapped))
             for r in range(world)]
    for p in procs:
        p.start()
    parts = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    parts.sort(key=lambda t: t[1])
    got = np.concatenate([p[2] for p in parts], axis=0)
    c = CASES[case]
    want = O.iterate(oracle_desc(c), make_grid(c), ITERS)
    assert got.tobytes() == want.tobytes()


def test_rowshard_geometry():
    shards = [RowShard(100, 8, r, 3, 2, 1) for r in range(3)]
    assert [(s.r0, s.r1) for s in shards] == [(0, 33), (33, 66), (66, 100)]
    assert [s.rows_above for s in shards] == [0, 2, 2]
    assert [s.rows_below for s in shards] == [1, 1, 0]
    assert shards[1].buffer_rows == 2 + 33 + 1
    with pytest.raises(ValueError):
        RowShard(4, 8, 0, 4, 2, 2).check()


def test_nccl_schedules_reject_temporal_blocking():
    """one launch of a TB > 1 descriptor advances TB generations,
    but the NCCL schedules only exchange N/S-deep halos per launch."""
    import pytest

    from paper_1511_02490_b200 import Stencil
    from paper_1511_02490_b200.distributed import RowShard, cuda_step, iterate_sharded_overlapped

    st = Stencil(op="heat", dtype="float32", load_path="strips", fused_iterations=4)
    with pytest.raises(ValueError, match="fused_iterations"):
        cuda_step(st, 32, 8)
    shard = RowShard(64, 32, 0, 2, 1, 1)
    a = torch.zeros((shard.buffer_rows, 32))
    with pytest.raises(ValueError, match="fused_iterations"):
        iterate_sharded_overlapped(a, a.clone(), shard, 3, st, 32, 8)
    cuda_step(Stencil(op="heat", dtype="float32"), 32, 8)  # one generation per launch: fine
