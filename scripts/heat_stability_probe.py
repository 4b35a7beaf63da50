"""Heat 16384^2 f32 x 100 generations, repeated: per-step time, SM clock,
power and throttle reasons (NVML every 10 ms) - is the config-3 variance
between bench runs power / clock behaviour or block choice?"""
import json
import sys
import threading
import time
from pathlib import Path

import pynvml
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1511_02490_b200 import Stencil  # noqa: E402

pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
st = Stencil(op="heat", dtype="float32", border="nearest")
n = 16384
a = torch.rand((n, n), device="cuda")
b = torch.empty_like(a)
for wc, wr in [(212, 4), (88, 8), (240, 4), (116, 6), (54, 16)]:
    st.iterate(a, b, 20, wc, wr)
    torch.cuda.synchronize()
    steps = []
    samples = []
    stop = threading.Event()

    def poll():
        while not stop.is_set():
            samples.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                            pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_MEM),
                            pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0,
                            pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)))
            stop.wait(0.01)

    t = threading.Thread(target=poll)
    t.start()
    for _ in range(8):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        st.iterate(a, b, 100, wc, wr)
        e1.record()
        e1.synchronize()
        steps.append(round(e0.elapsed_time(e1) / 100 * 1e3, 1))
    stop.set()
    t.join()
    sm = sorted(x[0] for x in samples)
    pw = sorted(x[2] for x in samples)
    reasons = sorted({r for x in samples for r in (("power_cap", 4), ("hw_slow", 8), ("sw_therm", 32), ("hw_therm", 64)) if x[3] & r[1]})
    print(json.dumps({"block": f"{wc}x{wr}", "us_per_gen": steps, "sm_mhz_median": sm[len(sm) // 2],
                      "mem_mhz": samples[len(samples) // 2][1], "power_w_median": pw[len(pw) // 2],
                      "power_w_max": pw[-1], "reasons": [r[0] for r in reasons]}), flush=True)
