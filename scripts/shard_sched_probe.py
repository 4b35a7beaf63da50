"""Cost of the row-shard NCCL schedule at one rank (sk_stencil_iterate_nccl:
interior + two boundary strips per generation, no exchange) against one pass
per generation, GoL 8192^2 i32 and heat 16384^2 f32 - the weak-scaling ceiling
of the schedule before NVLink time.  Prints one JSON line per workload."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1511_02490_b200 import Stencil  # noqa: E402
from paper_1511_02490_b200.distributed import RowShard, iterate_sharded_nccl  # noqa: E402

for op, dtype, H, W, border, (wc, wr) in [("gol", torch.int32, 8192, 8192, "pad", (36, 28)),
                                          ("heat", torch.float32, 16384, 16384, "nearest", (88, 8))]:
    st = Stencil(op=op, dtype={torch.int32: "int32", torch.float32: "float32"}[dtype], border=border)
    sh = RowShard(H, W, 0, 1, 1, 1)
    a = torch.zeros((sh.buffer_rows, W), dtype=dtype, device="cuda")
    a[1:1 + H] = (torch.rand((H, W), device="cuda") < 0.5).to(dtype)
    b = torch.zeros_like(a)
    x0 = a.clone()
    it = 20
    want = st.iterate(a[1:1 + H].clone(), torch.empty((H, W), dtype=dtype, device="cuda"), it, wc, wr).clone()
    got = iterate_sharded_nccl(a, b, sh, it, st, wc, wr)
    exact = bool(torch.equal(sh.owned(got), want))
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    res = {}
    for name, fn in (("one_pass", lambda: st.iterate(a[1:1 + H], b[1:1 + H], it, wc, wr)),
                     ("schedule", lambda: iterate_sharded_nccl(a, b, sh, it, st, wc, wr))):
        fn()
        torch.cuda.synchronize()
        e0, e1 = ev(), ev()
        e0.record()
        for _ in range(5):
            fn()
        e1.record()
        torch.cuda.synchronize()
        res[name] = e0.elapsed_time(e1) / (5 * it)
    print(json.dumps({"workload": op, "block": f"{wc}x{wr}", "one_pass_ms": round(res["one_pass"], 5),
                      "schedule_ms": round(res["schedule"], 5),
                      "one_pass_over_schedule": round(res["one_pass"] / res["schedule"], 4),
                      "bit_exact": exact}), flush=True)
