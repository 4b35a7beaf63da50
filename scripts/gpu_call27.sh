#!/usr/bin/env bash
cd "$(dirname "$0")/.."
O=gpurun_out/c28; mkdir -p $O
timeout 600 python -m pytest tests/test_div_const.py -q > $O/pytest_div.log 2>&1; echo "rc=$?" >> $O/pytest_div.log; tail -3 $O/pytest_div.log
timeout 600 python -m pytest tests/test_stencil_parity.py -q -k "boxmean or golden or ragged" > $O/pytest_box.log 2>&1; echo "rc=$?" >> $O/pytest_box.log; tail -2 $O/pytest_box.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_stencil -s 2 -c 1 -o $O/prof_boxmean python scripts/profile_pass.py boxmean float32 4096 4096 84 6 4 auto nearest > $O/ncu.log 2>&1
python3 - <<'PY'
import sys
sys.path.insert(0, '.')
import torch
from paper_1511_02490_b200 import Stencil
st = Stencil(op="boxmean", dtype="float32", north=5, south=1, east=3, west=0, border="nearest")
a = torch.rand((4096, 4096), device="cuda"); b = torch.empty_like(a)
best = None
for wc, wr in [(84, 6), (96, 8), (96, 4), (64, 8), (128, 4), (216, 4), (64, 4)]:
    ms = sorted(st.time(a, b, wc, wr, samples=30, warmup=3, flush_l2=True))
    m = sum(ms) / len(ms)
    print(f"boxmean(5,1,3,0) 4096^2 {wc}x{wr}: {m*1e3:.1f} us, {4096*4096/(m/1e3)/1e9:.1f} Gcells/s")
PY
