"""Exhaustive wc x wr sweep of the GENERATED synthetic kernels (wgtb gen-kernel,
results/generated/lib) on the fp32 datasets 512^2 .. 4096^2: every even size
with area <= 1024 (space.cpp:134-145), 2 warm-up + 5 timed launches (CUDA
events, L2 flushed before each sample), each size's output checked against
the scenario's gold output (itself checked against the generated C reference
on the two smaller grids).  Writes the reference's CSV formats
(datastore.cpp:18-19) plus contexts into results/generated/.
usage: python scripts/sweep_generated.py [samples]"""
import ctypes
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import numpy as np
import torch

from paper_1511_02490_b200 import _native as N
from paper_1511_02490_b200 import fill_host

GEN = ROOT / "results" / "generated"
KDIR = ROOT / "results" / "b200" / "descriptors" / "kernels"
SAMPLES = int(sys.argv[1]) if len(sys.argv) > 1 else 5
SIZES = [(c, r) for c in range(2, 513, 2) for r in range(2, 1024 // c + 1, 2)]
lib = N.lib()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
out_s = ["scenario_id,w_c,w_r,runtime_ms"]
out_r = ["scenario_id,w_c,w_r"]
out_c = ["scenario_id,device_max,kernel_max"]
log = []
for kj in sorted(KDIR.glob("synthetic-*.json")):
    k = json.loads(kj.read_text())
    name = k["name"]
    gen = ctypes.CDLL(str(GEN / "lib" / f"lib{name}.so"))
    table = (ctypes.c_void_p * 8)()
    assert gen.sk_gen_table(ctypes.byref(table)) == 0
    ref = ctypes.CDLL(str(GEN / "lib" / f"lib{name}_ref.so"))
    ref.gen_grid.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_long, ctypes.c_long, ctypes.c_int,
                             ctypes.c_float]
    d = N.sk_stencil_desc(op=0, dtype=N.SK_FLOAT32, north=k["north"], south=k["south"], east=k["east"],
                          west=k["west"], border_mode=N.SK_BORDER_NEAREST, pad_value=0.0)
    for side in (512, 1024, 2048, 4096):
        sid = f"NVIDIA-B200/{name}/{side}x{side}/FLOAT32-FLOAT32"
        t0 = time.time()
        host = np.empty((side, side), dtype=np.float32)
        fill_host(host, 1, 5)
        a = torch.from_numpy(host).cuda()
        b = torch.empty_like(a)
        gold = None
        mismatches = 0
        rows = []

        def launch(wc, wr):
            return lib.sk_stencil_launch_custom(ctypes.byref(d), ctypes.byref(table), a.data_ptr(), b.data_ptr(),
                                                side, side, side, side, 0, 0, wc, wr, None)

        for wc, wr in SIZES:
            rc = launch(wc, wr)
            if rc in (N.SK_REFUSED,):
                out_r.append(f"{sid},{wc},{wr}")
                continue
            if rc == N.SK_OVERSIZED:
                continue
            assert rc == 0, N.last_error()
            if gold is None:
                gold = b.clone()
                if side <= 1024:
                    want = np.empty_like(host)
                    ref.gen_grid(host.ctypes.data, want.ctypes.data, side, side, 1, 0.0)
                    assert gold.cpu().numpy().tobytes() == want.tobytes(), f"{sid}: gold != C reference"
            elif not torch.equal(b, gold):
                mismatches += 1
            launch(wc, wr)
            ts = []
            for _ in range(SAMPLES):
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                launch(wc, wr)
                e1.record()
                e1.synchronize()
                ts.append(e0.elapsed_time(e1))
            rows.append((wc, wr, sum(ts) / len(ts)))
        assert mismatches == 0, f"{sid}: {mismatches} sizes differ from the gold output"
        for wc, wr, ms in rows:
            out_s.append(f"{sid},{wc},{wr},{ms!r}")
        out_c.append(f"{sid},1024,1024")
        best = min(rows, key=lambda r: r[2])
        log.append(f"{sid}: {len(rows)} sizes in {time.time() - t0:.1f} s, oracle {best[0]}x{best[1]} "
                   f"{best[2] * 1e3:.1f} us, 0 gold mismatches")
        print(log[-1], flush=True)
(GEN / "samples.csv").write_text("\n".join(out_s) + "\n")
(GEN / "refused.csv").write_text("\n".join(out_r) + "\n")
(GEN / "contexts.csv").write_text("\n".join(out_c) + "\n")
(GEN / "collect.log").write_text("\n".join(log) + "\n")
