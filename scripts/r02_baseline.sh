#!/usr/bin/env bash
# Round-2 baseline evidence: GPU suite + ncu --set full of config 4's oracle
# block and of GoL at narrow (losing) block shapes.
cd "$(dirname "$0")/.."
O=gpurun_out/r02a; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" | tee -a $O/pytest_gpu.log
tail -3 $O/pytest_gpu.log
cap() { # name kernel-regex args...
  local n=$1 k=$2; shift 2
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 -o $O/$n python scripts/profile_pass.py "$@" > $O/$n.log 2>&1
  python scripts/ncu_digest.py $O/$n.ncu-rep > $O/${n}_digest.txt 2>/dev/null
  ncu -i $O/$n.ncu-rep --page raw --csv > $O/${n}_raw.csv 2>/dev/null
  ncu -i $O/$n.ncu-rep --page source --csv > $O/${n}_source.csv 2>/dev/null
  rm -f $O/$n.ncu-rep
}
cap boxmean5130_96x4 k_stencil boxmean float32 4096 4096 96 4 4 auto nearest
cap gol_2x2 k_stencil gol int32 8192 8192 2 2 4
cap gol_4x4 k_stencil gol int32 8192 8192 4 4 4
cap gol_2x64 k_stencil gol int32 8192 8192 2 64 4
cap gol_128x8 k_stencil gol int32 8192 8192 128 8 4
ls -la $O
