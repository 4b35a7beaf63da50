#!/usr/bin/env bash
# Round-2 ncu evidence: launch list of the bench's timed region at the tuned
# block (no sweep), and --set full captures of the dominant kernels: GoL at
# the bench's oracle block, config 4 at its oracle block, and GoL at the
# narrow (losing) blocks that explain the sweep's spread.
cd "$(dirname "$0")/.."
O=gpurun_out/${OUT:-r02ev}; mkdir -p $O
WC=${WC:-36}; WR=${WR:-28}
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file $O/launches_timed.csv \
  python bench.py --steps 2 --warmup 3 --wc $WC --wr $WR --no-cpu --no-e2e --no-temporal --no-configs > $O/ncu_bench.log 2>&1
echo "launch list rc=$?"
cap() { # name kernel-regex args...
  local n=$1 k=$2; shift 2
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 -o $O/$n python scripts/profile_pass.py "$@" > $O/$n.log 2>&1
  python scripts/ncu_digest.py $O/$n.ncu-rep > $O/${n}_digest.txt 2>/dev/null
  ncu -i $O/$n.ncu-rep --page raw --csv > $O/${n}_raw.csv 2>/dev/null
  ncu -i $O/$n.ncu-rep --page source --csv > $O/${n}_source.csv 2>/dev/null
  rm -f $O/$n.ncu-rep
}
cap gol_${WC}x${WR} k_stencil gol int32 8192 8192 $WC $WR 4
cap box_32x4 k_stencil boxmean float32 4096 4096 32 4 4 auto nearest
cap gol_2x2 k_stencil gol int32 8192 8192 2 2 4
cap gol_4x4 k_stencil gol int32 8192 8192 4 4 4
cap gol_2x64 k_stencil gol int32 8192 8192 2 64 4
cap heat_88x8 k_stencil heat float32 16384 16384 88 8 4 auto nearest
ls $O
