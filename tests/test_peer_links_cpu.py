"""Host-side wiring of the peer-memory halo exchange (no GPU needed): which
neighbour buffers and control blocks each rank's sk_halo_peers points at,
the north neighbour's row count (its south-halo offset), and the buffer-role
swap when a call passes (B, A) after an odd number of generations."""
from __future__ import annotations

import pytest

torch = pytest.importorskip("torch")

from paper_1511_02490_b200 import _native as N  # noqa: E402
from paper_1511_02490_b200.distributed import PeerLinks, RowShard, local_links  # noqa: E402


def ranks(world, H=50, W=8, n=1, s=2):
    shards = [RowShard(H, W, p, world, n, s) for p in range(world)]
    bufs = [(torch.zeros(sh.buffer_rows, W), torch.zeros(sh.buffer_rows, W), torch.zeros(8, dtype=torch.int64))
            for sh in shards]
    return shards, bufs


@pytest.mark.parametrize("world", [1, 2, 3, 5])
def test_local_links_point_at_neighbours(world):
    shards, bufs = ranks(world)
    links = local_links(bufs, shards)
    for p, ln in enumerate(links):
        q = ln.peers
        if p == 0:
            assert not q.north_a and not q.north_b and not q.north_control
        else:
            a, b, c = bufs[p - 1]
            assert (q.north_a, q.north_b, q.north_control) == (a.data_ptr(), b.data_ptr(), c.data_ptr())
            assert q.north_rows == shards[p - 1].rows
        if p == world - 1:
            assert not q.south_a and not q.south_b and not q.south_control
        else:
            a, b, c = bufs[p + 1]
            assert (q.south_a, q.south_b, q.south_control) == (a.data_ptr(), b.data_ptr(), c.data_ptr())
        assert ln.own == (bufs[p][0].data_ptr(), bufs[p][1].data_ptr())
        assert ln.control is bufs[p][2]


def test_peers_for_swaps_roles_with_the_buffers():
    shards, bufs = ranks(3)
    ln = local_links(bufs, shards)[1]
    a, b, _ = bufs[1]
    same = ln.peers_for(a, b)
    assert same is ln.peers
    sw = ln.peers_for(b, a)
    q = ln.peers
    assert (sw.north_a, sw.north_b, sw.south_a, sw.south_b) == (q.north_b, q.north_a, q.south_b, q.south_a)
    assert (sw.north_control, sw.south_control, sw.north_rows) == (q.north_control, q.south_control,
                                                                   q.north_rows)
    with pytest.raises(ValueError):
        ln.peers_for(a, torch.zeros_like(b))


def test_peer_struct_layout_matches_header():
    """sk_halo_peers / sk_ipc_handle field order and sizes as declared in
    include/sk_stencil.h (seven 8-byte fields; 64-byte handle + offset)."""
    assert [f[0] for f in N.sk_halo_peers._fields_] == [
        "north_a", "north_b", "south_a", "south_b", "north_control", "south_control", "north_rows"]
    assert N.ctypes.sizeof(N.sk_halo_peers) == 56
    assert N.ctypes.sizeof(N.sk_ipc_handle) == 72
    text = N.HEADER_PATH.read_text()
    assert "#define SK_HALO_CONTROL_BYTES 64" in text and N.SK_HALO_CONTROL_BYTES == 64
    assert isinstance(PeerLinks(N.sk_halo_peers(), None).epoch, int)
