"""Exhaustive wc x wr sweep of the GENERATED synthetic kernels (wgtb gen-kernel
-> scripts/gen_study_kernels.sh -> results/generated/lib): all 40 synthetic
kernels of the study on the fp32 datasets 512^2 .. 8192^2; every even size with
area <= 1024 (space.cpp:134-145); per size one validation launch (the output
must equal the scenario's gold output, itself equal to the generated C
reference on the two smaller grids), 2 warm-ups and `samples` timed launches
(CUDA events; before each sample 2 x L2 is written then read back, so the
timed pass carries no write-back debt - DESIGN.md §4.4d).  One CSV line per
observation in the reference's formats (datastore.cpp:18-19) plus contexts,
checkpointed after every scenario and resumable (completed scenarios in the
output directory are skipped).
usage: python scripts/sweep_generated.py OUT_DIR [samples] [max_seconds]"""
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
OUT = Path(sys.argv[1]) if len(sys.argv) > 1 else GEN
SAMPLES = int(sys.argv[2]) if len(sys.argv) > 2 else 5
BUDGET = float(sys.argv[3]) if len(sys.argv) > 3 else 1e9
SIDES = (512, 1024, 2048, 4096, 8192)
SIZES = [(c, r) for c in range(2, 513, 2) for r in range(2, 1024 // c + 1, 2)]
lib = N.lib()
props = N.sk_device_props()
N.check(lib.sk_device_features(0, ctypes.byref(props)), "sk_device_features")
scrub = torch.empty(2 * 126 * (1 << 20), dtype=torch.uint8, device="cuda")
OUT.mkdir(parents=True, exist_ok=True)
files = {"samples": (OUT / "samples.csv", "scenario_id,w_c,w_r,runtime_ms"),
         "refused": (OUT / "refused.csv", "scenario_id,w_c,w_r"),
         "contexts": (OUT / "contexts.csv", "scenario_id,device_max,kernel_max")}
for p, header in files.values():
    if not p.exists():
        p.write_text(header + "\n")
done = {ln.split(",", 1)[0] for ln in files["contexts"][0].read_text().splitlines()[1:]}
t_start = time.time()


def scrubbed():
    scrub.fill_(1)
    return int(scrub.view(torch.int64).sum().item() & 1)  # read it back: clean lines only


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
    for side in SIDES:
        sid = f"{props.name.decode().replace(' ', '-')}/{name}/{side}x{side}/FLOAT32-FLOAT32"
        if sid in done:
            continue
        if time.time() - t_start > BUDGET:
            print("budget reached", flush=True)
            sys.exit(0)
        t0 = time.time()
        host = np.empty((side, side), dtype=np.float32)
        fill_host(host, 1, 5)
        a = torch.from_numpy(host).cuda()
        b = torch.empty_like(a)
        gold = None
        rows, refused, mismatched = [], [], []
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * SAMPLES)]

        def launch(wc, wr):
            return lib.sk_stencil_launch_custom(ctypes.byref(d), ctypes.byref(table), a.data_ptr(), b.data_ptr(),
                                                side, side, side, side, 0, 0, wc, wr, None)

        for wc, wr in SIZES:
            rc = launch(wc, wr)
            if rc == N.SK_REFUSED:
                refused.append((wc, wr))
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
                mismatched.append((wc, wr))  # rejected: never timed, recorded as refused
                refused.append((wc, wr))
                continue
            for _ in range(2):
                launch(wc, wr)
            for i in range(SAMPLES):
                scrubbed()
                ev[2 * i].record()
                launch(wc, wr)
                ev[2 * i + 1].record()
            torch.cuda.synchronize()
            rows.append((wc, wr, [ev[2 * i].elapsed_time(ev[2 * i + 1]) for i in range(SAMPLES)]))
        with files["samples"][0].open("a") as f:
            for wc, wr, ts in rows:
                for t in ts:
                    f.write(f"{sid},{wc},{wr},{max(t, 1e-6)!r}\n")
        with files["refused"][0].open("a") as f:
            for wc, wr in refused:
                f.write(f"{sid},{wc},{wr}\n")
        with files["contexts"][0].open("a") as f:
            f.write(f"{sid},1024,1024\n")
        best = min(rows, key=lambda r: sum(r[2]))
        msg = (f"{sid}: {len(rows)} sizes in {time.time() - t0:.1f} s, oracle {best[0]}x{best[1]} "
               f"{sum(best[2]) / SAMPLES * 1e3:.1f} us, {len(mismatched)} gold mismatches")
        with (OUT / "collect.log").open("a") as f:
            f.write(msg + "\n")
        print(msg, flush=True)
