"""Peer-memory halo exchange fused into the boundary-strip kernel
(csrc/stencil/halo.cuh, sk_stencil_iterate_peer).

Each gpurun box has one GPU, so the P "ranks" of the single-process tests
live in one process, each with its own buffers, control block and CUDA
stream; their peer pointers are the neighbours' tensors.  The device-side
protocol (strip pass stores into the neighbour's halo, last block publishes
the generation, the neighbour's next strip pass acquires it) is exactly the
multi-GPU one - only the mapping differs (IPC over NVLink across devices).
Launches of all ranks are enqueued round-robin from one host thread, so no
rank's host code ever waits for another's: the ordering is the device
flags'.  Results must be bit-identical to the undivided CPU oracle.

The two-process test maps the neighbour's buffers with CUDA IPC handles
(sk_ipc_export / sk_ipc_import) as a multi-GPU run does.  Both schedules are
covered: the strips + interior kernels (the default) and the opt-in one-pass
kernel with the exchange fused into its boundary tile-rows (forced here on
small grids)."""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

import oracle_lib as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_1511_02490_b200 import Stencil  # noqa: E402
from paper_1511_02490_b200.distributed import (RowShard, iterate_sharded_peer, local_links,  # noqa: E402
                                               new_control)

ROOT = Path(__file__).resolve().parent.parent
TDT = {"int32": torch.int32, "float32": torch.float32, "float64": torch.float64}


def grid(op, dtype, shape, seed):
    rng = np.random.default_rng(seed)
    if op == "gol":
        return (rng.random(shape) < 0.4).astype(dtype)
    if dtype == "int32":
        return rng.integers(-1000, 1000, size=shape).astype(np.int32)
    return (2 * rng.random(shape) - 1).astype(dtype)


def run_ranks(st, x, world, iterations, wc=32, wr=8, calls=1):
    """P logical ranks on one GPU; `calls` consecutive iterate calls (the
    epoch carries across them).  Returns the gathered grid.  Temporally
    blocked stencils (TB generations per exchange) get TB-deep halos."""
    H, W = x.shape
    depth = max(1, st.fused_iterations)
    n, s = depth * st.north, depth * st.south
    shards = [RowShard(H, W, p, world, n, s) for p in range(world)]
    bufs, streams = [], []
    for sh in shards:
        a = torch.zeros((sh.buffer_rows, W), dtype=TDT[str(x.dtype)], device="cuda")
        a[n:n + sh.rows] = torch.from_numpy(np.ascontiguousarray(x[sh.r0:sh.r1])).cuda()
        bufs.append((a, torch.zeros_like(a), new_control()))
        streams.append(torch.cuda.Stream())
    torch.cuda.synchronize()
    links = local_links(bufs, shards)
    cur = [(a, b) for a, b, _ in bufs]
    per_call = [iterations // calls + (1 if c < iterations % calls else 0) for c in range(calls)]
    for its in per_call:
        for p, sh in enumerate(shards):  # round-robin enqueue, no host waits
            a, b = cur[p]
            res = iterate_sharded_peer(a, b, sh, its, st, wc, wr, links[p], stream=streams[p])
            cur[p] = (res, b if res is a else a)
    torch.cuda.synchronize()
    return np.concatenate([sh.owned(cur[p][0]).cpu().numpy() for p, sh in enumerate(shards)])


CASES = [
    ("heat", "float32", (1, 1, 1, 1), "nearest", 0.0),
    ("five_point", "float64", (1, 1, 1, 1), "pad", 0.5),
    ("gol", "int32", (1, 1, 1, 1), "pad", 0.0),
    ("boxmean", "float32", (5, 1, 3, 0), "nearest", 0.0),
    ("gaussian", "int32", (2, 2, 2, 2), "pad", 3.0),
    ("sobel", "float32", (1, 1, 1, 1), "nearest", 0.0),
]


@pytest.fixture(params=["auto", "fused"])
def schedule(request, monkeypatch):
    """auto: the strips + interior schedule (the default);
    fused: the opt-in one-pass kernel with the exchange in its boundary
    tile-rows - small grids, so the ranks' persistent grids never starve
    each other of SMs on the shared GPU."""
    if request.param == "fused":
        monkeypatch.setenv("SK_PEER_SCHEDULE", "fused")
        monkeypatch.setenv("SK_PEER_ALLOW_SHARED", "1")
    else:
        monkeypatch.delenv("SK_PEER_SCHEDULE", raising=False)
    return request.param


@pytest.mark.parametrize("op,dtype,borders,border,pad", CASES)
@pytest.mark.parametrize("world", [2, 3])
def test_peer_exchange_vs_oracle(op, dtype, borders, border, pad, world, schedule):
    n, s, e, w = borders
    st = Stencil(op=op, dtype=dtype, north=n, south=s, east=e, west=w, border=border,
                 pad_value=pad)
    x = grid(op, dtype, (61, 150), seed=world * 11 + n)
    iters = 7
    got = run_ranks(st, x, world, iters)
    want = O.iterate(O.desc_from_stencil(st), x, iters)
    assert got.tobytes() == want.tobytes()


@pytest.mark.parametrize("world", [2, 4])
def test_peer_exchange_epochs_and_thin_shards(world, schedule):
    """Several iterate calls back to back (the epoch counter carries the
    flag protocol across calls) and shards only a little taller than the
    strips (h < 2m: the top strip owns every row)."""
    st = Stencil(op="boxmean", dtype="float32", north=5, south=1, east=3, west=0,
                 border="nearest")
    x = grid("boxmean", "float32", (world * 7, 90), seed=world)
    got = run_ranks(st, x, world, 10, wc=16, wr=4, calls=3)
    want = O.iterate(O.desc_from_stencil(st), x, 10)
    assert got.tobytes() == want.tobytes()


def test_peer_exchange_config3_shape():
    """Heat, 4 ranks over a 4096 x 4096 grid, 20 generations: the gathered
    result equals the undivided executor's (a size-independent property)."""
    from paper_1511_02490_b200 import fill_host

    host = np.empty((4096, 4096), dtype=np.float32)
    fill_host(host, 1, 3)
    st = Stencil(op="heat", dtype="float32", border="nearest")
    a = torch.from_numpy(host).cuda()
    want = st.iterate(a.clone(), torch.empty_like(a), 20, 64, 8).cpu().numpy()
    got = run_ranks(st, host, 4, 20, wc=64, wr=8)
    assert got.tobytes() == want.tobytes()


def test_peer_rejects_per_cell_fused_and_bitplane():
    for st in (Stencil(op="heat", dtype="float32", fused_iterations=4, load_path="tma"),
               Stencil(op="gol", dtype="int32", fused_iterations=8)):
        with pytest.raises(Exception):
            run_ranks(st, grid(st.op, st.dtype, (120, 40), 1), 2, 3)


@pytest.mark.parametrize("op,dtype,border,pad", [("heat", "float32", "nearest", 0.0),
                                                 ("five_point", "int32", "pad", 7.0),
                                                 ("heat", "float64", "pad", 0.25)])
@pytest.mark.parametrize("tb,world", [(4, 2), (8, 3), (5, 2)])
def test_peer_exchange_temporal_blocking(op, dtype, border, pad, tb, world):
    """Register-strip path, TB generations per exchange (TB-deep halos, the
    strips / put / interior schedule of sk_stencil_iterate_peer), over three
    consecutive calls whose generation counts are not multiples of TB."""
    st = Stencil(op=op, dtype=dtype, border=border, pad_value=pad, load_path="strips",
                 fused_iterations=tb)
    x = grid(op, dtype, (world * 70, 333), seed=tb * 10 + world)
    got = run_ranks(st, x, world, 29, wc=32, wr=8, calls=3)
    want = O.iterate(O.desc_from_stencil(st), x, 29)
    assert got.tobytes() == want.tobytes()


def test_peer_exchange_two_processes_ipc():
    """Two processes, buffers mapped with CUDA IPC handles (both on cuda:0
    here; across GPUs the same handles map over NVLink)."""
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT="29613",
               PYTHONPATH=str(ROOT) + os.pathsep + str(ROOT / "tests"))
    out = subprocess.run([sys.executable, str(ROOT / "tests" / "peer_ipc_worker.py")],
                         env=env, capture_output=True, text=True, timeout=240)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "peer-ipc: ok" in out.stdout
