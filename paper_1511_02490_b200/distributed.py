"""Row-block decomposition of iterated stencils over P ranks (north-star
subsystem 5).

Rank p owns global rows [p*H/P, (p+1)*H/P) and keeps them in a buffer of
N + rows + S rows: N north-halo rows, the owned rows, S south-halo rows.
Per iteration, inside one batched P2P group:

    send my first S owned rows  -> p-1   (its south halo)
    recv my north halo (N rows) <- p-1
    send my last N owned rows   -> p+1   (its north halo)
    recv my south halo (S rows) <- p+1

Row-major storage makes every message a contiguous slice (no packing).  The
global edges (rank 0's north, rank P-1's south) have no halo: the launch
passes rows_above = 0 / rows_below = 0 there and the executor applies the
border mode (pad or nearest) exactly as the single-GPU pass does, so the
decomposed run is bit-identical to the undivided one.

Transport is torch.distributed point-to-point (NCCL over NVLink on B200,
gloo on CPU for the multi-process tests).  The per-iteration compute is a
callable so the same exchange logic drives the CUDA executor in production
and the CPU oracle in tests.

The peer transport (`iterate_sharded_peer`, C-ABI sk_stencil_iterate_peer)
fuses the exchange into the boundary-strip kernel instead: the strips store
the rows a neighbour needs straight into its halo through a peer mapping of
its buffers (CUDA IPC over NVLink / NVSwitch) and publish an arrival flag the
neighbour's next strip pass acquires on the device - no NCCL call and no host
synchronisation per generation.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from typing import Callable

import torch
import torch.distributed as dist


@dataclass(frozen=True)
class RowShard:
    height: int   # global rows
    width: int
    rank: int
    world: int
    north: int
    south: int

    @property
    def r0(self) -> int:
        return self.rank * self.height // self.world

    @property
    def r1(self) -> int:
        return (self.rank + 1) * self.height // self.world

    @property
    def rows(self) -> int:
        return self.r1 - self.r0

    @property
    def rows_above(self) -> int:
        """Halo rows that hold real data above the owned rows."""
        return self.north if self.rank > 0 else 0

    @property
    def rows_below(self) -> int:
        return self.south if self.rank < self.world - 1 else 0

    @property
    def buffer_rows(self) -> int:
        return self.north + self.rows + self.south

    def check(self) -> None:
        if self.rows < max(self.north, self.south, 1):
            raise ValueError(f"rank {self.rank} owns {self.rows} rows; halos need "
                             f">= max(N={self.north}, S={self.south})")

    def owned(self, buf: torch.Tensor) -> torch.Tensor:
        return buf[self.north:self.north + self.rows]


def _staged_exchange(buf: torch.Tensor, shard: RowShard, group=None) -> None:
    """gloo cannot move CUDA tensors: stage the halo slices through host
    memory (used only to exercise the multi-rank path on a single GPU)."""
    cpu = torch.empty((shard.buffer_rows, buf.shape[1]), dtype=buf.dtype)
    n, s, h = shard.north, shard.south, shard.rows
    cpu[n:n + h].copy_(buf[n:n + h])
    exchange_halos(cpu, shard, group)
    if shard.rank > 0 and n:
        buf[0:n].copy_(cpu[0:n])
    if shard.rank < shard.world - 1 and s:
        buf[n + h:n + h + s].copy_(cpu[n + h:n + h + s])


def exchange_halos(buf: torch.Tensor, shard: RowShard, group=None) -> None:
    """Fill the north/south halo rows of `buf` from the neighbouring ranks."""
    if buf.is_cuda and dist.get_backend(group) == "gloo":
        _staged_exchange(buf, shard, group)
        return
    n, s, h = shard.north, shard.south, shard.rows
    ops = []
    if shard.rank > 0:
        prev = shard.rank - 1
        if s:
            ops.append(dist.P2POp(dist.isend, buf[n:n + s], prev, group))
        if n:
            ops.append(dist.P2POp(dist.irecv, buf[0:n], prev, group))
    if shard.rank < shard.world - 1:
        nxt = shard.rank + 1
        if n:
            ops.append(dist.P2POp(dist.isend, buf[n + h - n:n + h], nxt, group))
        if s:
            ops.append(dist.P2POp(dist.irecv, buf[n + h:n + h + s], nxt, group))
    if ops:
        for work in dist.batch_isend_irecv(ops):
            work.wait()


StepFn = Callable[[torch.Tensor, torch.Tensor, RowShard], None]
"""step(src_buf, dst_buf, shard): one stencil pass from src's owned rows (with
shard.rows_above / rows_below halo rows readable around them) into dst's
owned rows."""


def iterate_sharded(a: torch.Tensor, b: torch.Tensor, shard: RowShard, iterations: int,
                    step: StepFn, group=None) -> torch.Tensor:
    """`iterations` exchange+pass rounds ping-ponging a/b; returns the buffer
    holding the result (owned rows are shard.owned(result))."""
    shard.check()
    src, dst = a, b
    for _ in range(iterations):
        if shard.world > 1:
            exchange_halos(src, shard, group)
        step(src, dst, shard)
        src, dst = dst, src
    return src


def _one_generation_per_launch(stencil) -> None:
    """The NCCL schedules exchange N/S-deep halos once per launch, so a
    launch must advance exactly one generation: a temporally blocked
    descriptor (TB > 1 generations per launch) would read rows beyond the
    halo as border and silently change the result.  (The peer schedule,
    sk_stencil_iterate_peer, runs TB > 1 on the strip path with TB-deep
    halos.)"""
    tb = int(getattr(stencil.desc, "fused_iterations", 0)) if hasattr(stencil, "desc") else 0
    if tb > 1:
        raise ValueError(f"fused_iterations={tb}: the NCCL row-shard schedule needs one "
                         "generation per launch (use iterate_sharded_peer for TB > 1)")


def cuda_step(stencil, wc: int, wr: int) -> StepFn:
    """Production step: one sm_100a executor launch on the current stream."""
    _one_generation_per_launch(stencil)

    def step(src: torch.Tensor, dst: torch.Tensor, shard: RowShard) -> None:
        stencil(src[shard.north:], dst[shard.north:], wc, wr, rows_above=shard.rows_above,
                rows_below=shard.rows_below, height=shard.rows)

    return step


def iterate_sharded_overlapped(a: torch.Tensor, b: torch.Tensor, shard: RowShard,
                               iterations: int, stencil, wc: int, wr: int,
                               group=None) -> torch.Tensor:
    """CUDA executor with the halo exchange hidden behind the interior.

    Per generation (src -> dst) on the compute stream: the boundary strips
    are computed first.  Each strip is m = max(N, S) rows deep, because it
    must hold both the rows that read a halo (the first N / last S owned
    rows) and the rows the neighbour needs next (the first S rows go to p-1,
    the last N rows to p+1).  The exchange of dst's new boundary rows then
    runs on a communication stream while the interior rows [m, rows - m),
    which read only owned rows of src, are computed.  The next generation's
    boundary strips wait for that exchange.  Bit-identical to
    iterate_sharded."""
    shard.check()
    _one_generation_per_launch(stencil)
    n, s, h = shard.north, shard.south, shard.rows
    m = max(n, s)
    if h < 2 * max(m, 1) or shard.world == 1:
        return iterate_sharded(a, b, shard, iterations, cuda_step(stencil, wc, wr), group)

    def rows(src, dst, r0, r1):
        stencil(src[n + r0:], dst[n + r0:], wc, wr,
                rows_above=min(n, r0 + shard.rows_above), rows_below=min(s, h - r1 + shard.rows_below),
                height=r1 - r0)

    exchange_halos(a, shard, group)  # initial halos of the input
    src, dst = a, b
    if not a.is_cuda:
        # Host tensors (the multi-process CPU tests): the same schedule run
        # serially in its worst-case order - the exchange completes before
        # the interior is computed - so a strip that misses a row the
        # neighbour needs shows up as a wrong halo.
        for _ in range(iterations):
            rows(src, dst, 0, m)
            rows(src, dst, h - m, h)
            exchange_halos(dst, shard, group)
            if h - 2 * m > 0:
                rows(src, dst, m, h - m)
            src, dst = dst, src
        return src
    compute = torch.cuda.current_stream()
    comm = torch.cuda.Stream()
    exchanged = torch.cuda.Event()
    for _ in range(iterations):
        rows(src, dst, 0, m)             # top strip: reads the north halo, feeds p-1
        rows(src, dst, h - m, h)         # bottom strip: reads the south halo, feeds p+1
        strips = torch.cuda.Event()
        strips.record(compute)
        with torch.cuda.stream(comm):
            comm.wait_event(strips)
            exchange_halos(dst, shard, group)
            exchanged.record(comm)
        if h - 2 * m > 0:
            rows(src, dst, m, h - m)     # interior, concurrent with the exchange
        compute.wait_event(exchanged)
        src, dst = dst, src
    return src


def scatter_rows(full: torch.Tensor, shard: RowShard) -> torch.Tensor:
    """Buffer for `shard` initialised from the global grid (halos zero)."""
    buf = torch.zeros((shard.buffer_rows, shard.width), dtype=full.dtype, device=full.device)
    buf[shard.north:shard.north + shard.rows] = full[shard.r0:shard.r1]
    return buf


# ------------------------------------------------------------ peer transport
@dataclass
class PeerLinks:
    """What one rank needs for sk_stencil_iterate_peer: the neighbours' A/B
    buffers and control blocks mapped into this process, this rank's own
    control block (zeroed; the neighbours write its arrival flags) and the
    epoch counter all ranks advance in lockstep."""
    peers: object                      # _native.sk_halo_peers
    control: torch.Tensor              # SK_HALO_CONTROL_BYTES of device memory
    own: tuple = (0, 0)                # this rank's (A, B) data pointers as registered
    epoch: int = 0
    imported: list = field(default_factory=list)  # IPC mappings to close

    def peers_for(self, a: torch.Tensor, b: torch.Tensor):
        """The peer struct for a call on (a, b): every rank ping-pongs in
        lockstep, so when this rank passes its buffers swapped (an odd
        iteration count left the result in B) so do its neighbours."""
        from . import _native as N

        pa, pb = a.data_ptr(), b.data_ptr()
        if (pa, pb) == self.own:
            return self.peers
        if (pb, pa) != self.own:
            raise ValueError("iterate_sharded_peer: a/b are not the buffers the links were made for")
        q = self.peers
        return N.sk_halo_peers(q.north_b, q.north_a, q.south_b, q.south_a, q.north_control,
                               q.south_control, q.north_rows)

    def close(self) -> None:
        from . import _native as N

        for ptr in self.imported:
            N.lib().sk_ipc_close(ptr)
        self.imported.clear()


def new_control(device=None) -> torch.Tensor:
    from . import _native as N

    return torch.zeros(N.SK_HALO_CONTROL_BYTES // 8, dtype=torch.int64,
                       device=device or torch.device("cuda"))


def local_links(bufs: list, shards: list) -> list:
    """Links for P "ranks" that live in one process (one stream each): the
    neighbours' tensors are addressed directly.  bufs[p] = (a, b, control)."""
    from . import _native as N

    links = []
    for p, sh in enumerate(shards):
        peers = N.sk_halo_peers()
        if p > 0:
            a, b, c = bufs[p - 1]
            peers.north_a, peers.north_b, peers.north_control = a.data_ptr(), b.data_ptr(), c.data_ptr()
            peers.north_rows = shards[p - 1].rows
        if p < len(shards) - 1:
            a, b, c = bufs[p + 1]
            peers.south_a, peers.south_b, peers.south_control = a.data_ptr(), b.data_ptr(), c.data_ptr()
        links.append(PeerLinks(peers, bufs[p][2], (bufs[p][0].data_ptr(), bufs[p][1].data_ptr())))
    return links


def connect_peers(a: torch.Tensor, b: torch.Tensor, control: torch.Tensor, shard: RowShard,
                  group=None) -> PeerLinks:
    """Multi-process links: every rank exports IPC handles of its A, B and
    control block, all-gathers them (any backend), and maps its neighbours'.
    The control blocks are zero before the barrier that ends this call."""
    from . import _native as N

    torch.cuda.synchronize()

    def export(t):
        h = N.sk_ipc_handle()
        N.check(N.lib().sk_ipc_export(t.data_ptr(), ctypes.byref(h)), "sk_ipc_export")
        return bytes(h.handle), int(h.offset)

    mine = {"a": export(a), "b": export(b), "c": export(control), "rows": shard.rows}
    every = [None] * shard.world
    dist.all_gather_object(every, mine, group=group)

    links = PeerLinks(N.sk_halo_peers(), control, (a.data_ptr(), b.data_ptr()))

    def imp(entry):
        h = N.sk_ipc_handle()
        ctypes.memmove(h.handle, entry[0], len(entry[0]))
        h.offset = entry[1]
        ptr = ctypes.c_void_p()
        N.check(N.lib().sk_ipc_import(ctypes.byref(h), ctypes.byref(ptr)), "sk_ipc_import")
        links.imported.append(ptr.value)
        return ptr.value

    if shard.rank > 0:
        e = every[shard.rank - 1]
        links.peers.north_a, links.peers.north_b = imp(e["a"]), imp(e["b"])
        links.peers.north_control = imp(e["c"])
        links.peers.north_rows = e["rows"]
    if shard.rank < shard.world - 1:
        e = every[shard.rank + 1]
        links.peers.south_a, links.peers.south_b = imp(e["a"]), imp(e["b"])
        links.peers.south_control = imp(e["c"])
    dist.barrier(group=group)
    return links


def nccl_comm_ptr(group=None) -> int:
    """The raw ncclComm_t of torch's NCCL process group (for the C-ABI)."""
    pg = group or dist.distributed_c10d._get_default_group()
    return int(pg._get_backend(torch.device("cuda"))._comm_ptr())


def iterate_sharded_nccl(a: torch.Tensor, b: torch.Tensor, shard: RowShard, iterations: int,
                         stencil, wc: int, wr: int, comm: int | None = None, stream=None) -> torch.Tensor:
    """`iterations` generations through the C-ABI NCCL schedule
    (sk_stencil_iterate_nccl): ncclSend/ncclRecv of the halo rows on the
    library's exchange stream behind the interior pass, then the boundary
    strips.  `a` / `b` are the shard's N + rows + S row buffers; `comm` is a
    raw ncclComm_t (default: torch's NCCL group).  Returns the buffer holding
    the result; bit-identical to iterate_sharded."""
    from . import _native as N

    shard.check()
    _one_generation_per_launch(stencil)
    if shard.world > 1 and comm is None:
        comm = nccl_comm_ptr()
    s = (stream or torch.cuda.current_stream(a.device)).cuda_stream
    in_b = ctypes.c_int32(0)
    rc = N.lib().sk_stencil_iterate_nccl(ctypes.byref(stencil.desc), a.data_ptr(), b.data_ptr(), shard.width,
                                         shard.rows, a.stride(0), iterations, wc, wr, comm or None,
                                         shard.rank, shard.world, s or None, ctypes.byref(in_b))
    if rc:
        raise N.NativeError(rc, "sk_stencil_iterate_nccl", N.last_error())
    return b if in_b.value else a


def iterate_sharded_peer(a: torch.Tensor, b: torch.Tensor, shard: RowShard, iterations: int,
                         stencil, wc: int, wr: int, links: PeerLinks, stream=None) -> torch.Tensor:
    """`iterations` generations with the halo exchange fused into the
    boundary-strip kernel (sk_stencil_iterate_peer).  `a` / `b` are the
    shard's N + rows + S row buffers; returns the one holding the result.
    Bit-identical to iterate_sharded."""
    from . import _native as N

    shard.check()
    s = (stream or torch.cuda.current_stream(a.device)).cuda_stream
    epoch = ctypes.c_int64(links.epoch)
    in_b = ctypes.c_int32(0)
    peers = links.peers_for(a, b)
    rc = N.lib().sk_stencil_iterate_peer(ctypes.byref(stencil.desc), a.data_ptr(), b.data_ptr(),
                                         shard.width, shard.rows, a.stride(0), iterations, wc, wr,
                                         ctypes.byref(peers), links.control.data_ptr(),
                                         ctypes.byref(epoch), s or None, ctypes.byref(in_b))
    if rc:
        stencil._raise(rc, "sk_stencil_iterate_peer", wc, wr)
    links.epoch = epoch.value
    return b if in_b.value else a
