"""Single-process repro of the multi-rank boxmean mismatch: one pass per
shard with halos vs the oracle on the full grid."""
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
import numpy as np, torch
import oracle_lib as O
from paper_1511_02490_b200 import Stencil
from paper_1511_02490_b200.distributed import RowShard, scatter_rows

H, W = 203, 264
rng = np.random.default_rng(5)
full = rng.random((H, W)).astype(np.float32)
for borders in [(3, 2, 1, 0), (3, 2, 1, 2), (2, 2, 1, 1), (1, 1, 1, 1), (3, 3, 0, 0), (2, 1, 0, 0)]:
    n, s, e, w = borders
    for path in ("auto", "explicit"):
        st = Stencil(op="boxmean", dtype="float32", north=n, south=s, east=e, west=w, border="nearest", load_path=path)
        want = O.iterate(O.desc_from_stencil(st), full, 1)
        for world in (2, 3):
            for rank in range(world):
                sh = RowShard(H, W, rank, world, n, s)
                buf = torch.zeros((sh.buffer_rows, W), dtype=torch.float32, device="cuda")
                lo = sh.r0 - sh.rows_above
                hi = sh.r1 + sh.rows_below
                buf[n - sh.rows_above:n + sh.rows + sh.rows_below] = torch.from_numpy(full[lo:hi]).cuda()
                out = torch.zeros_like(buf)
                for wc, wr in ((32, 4), (16, 8)):
                    st(buf[n:], out[n:], wc, wr, rows_above=sh.rows_above, rows_below=sh.rows_below, height=sh.rows)
                    torch.cuda.synchronize()
                    got = sh.owned(out).cpu().numpy()
                    ref = want[sh.r0:sh.r1]
                    bad = np.argwhere(got != ref)
                    if len(bad):
                        print(f"{borders} {path} world={world} rank={rank} {wc}x{wr}: {len(bad)} bad, first {bad[:4].tolist()} rows={sh.rows}")
print("done")
