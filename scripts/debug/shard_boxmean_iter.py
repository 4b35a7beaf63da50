"""Single-process emulation of the row-sharded iteration (manual halo copies)."""
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
import numpy as np, torch
import oracle_lib as O
from paper_1511_02490_b200 import Stencil
from paper_1511_02490_b200.distributed import RowShard, scatter_rows

H, W, iters = 203, 264, 9
rng = np.random.default_rng(5)
full = rng.random((H, W)).astype(np.float32)
for borders in [(3, 2, 1, 0), (1, 1, 1, 1), (2, 2, 1, 0)]:
    n, s, e, w = borders
    st = Stencil(op="boxmean", dtype="float32", north=n, south=s, east=e, west=w, border="nearest")
    d = O.desc_from_stencil(st)
    for it in range(1, iters + 1):
        want = O.iterate(d, full, it)
        a = torch.from_numpy(full).cuda(); b = torch.empty_like(a)
        g1 = st.iterate(a, b, it, 32, 4).cpu().numpy()
        # sharded emulation
        world = 2
        shards = [RowShard(H, W, r, world, n, s) for r in range(world)]
        bufs = [[scatter_rows(torch.from_numpy(full).cuda(), sh), None] for sh in shards]
        for bb in bufs: bb[1] = torch.zeros_like(bb[0])
        cur = 0
        for _ in range(it):
            # exchange
            for r, sh in enumerate(shards):
                src = bufs[r][cur]
                if r > 0:
                    p = bufs[r - 1][cur]; ps = shards[r - 1]
                    src[0:n] = p[n + ps.rows - n:n + ps.rows]
                if r < world - 1:
                    q = bufs[r + 1][cur]
                    src[n + sh.rows:n + sh.rows + s] = q[n:n + s]
            for r, sh in enumerate(shards):
                src, dst = bufs[r][cur], bufs[r][1 - cur]
                st(src[n:], dst[n:], 32, 4, rows_above=sh.rows_above, rows_below=sh.rows_below, height=sh.rows)
            cur = 1 - cur
        torch.cuda.synchronize()
        got = np.concatenate([sh.owned(bufs[r][cur]).cpu().numpy() for r, sh in enumerate(shards)])
        print(borders, it, "single==oracle", (g1 == want).all(), "sharded==oracle", (got == want).all(),
              "bad rows", sorted(set(np.argwhere(got != want)[:, 0].tolist()))[:10])
