#!/usr/bin/env bash
# Round-1 evidence on one B200 (run under gpurun): GPU tests, the bench line,
# the ncu launch list of the bench command, one ncu --set full capture of the
# top kernel at the tuned block, and the BASELINE config-3/-4 measurements.
set -x
cd "$(dirname "$0")/.."
O=gpurun_out/r01
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt
timeout 900 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err
BLK=$(python -c "import json;d=json.load(open('$O/bench.json'));print(d['config']['block'].replace('x',' '))")
set -- $BLK
WC=$1; WR=$2
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $O/launches.csv \
  python bench.py --steps 1 --warmup 3 --wc $WC --wr $WR --no-e2e --no-cpu > $O/bench_under_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_stencil_tma -s 2 -c 1 \
  -o $O/prof_gol_${WC}x${WR} python scripts/profile_pass.py gol int32 8192 8192 $WC $WR 4 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none -k regex:k_stencil_tma -s 2 -c 1 \
  -o $O/prof_gol_32x4 python scripts/profile_pass.py gol int32 8192 8192 32 4 4 > /dev/null 2>&1
# config 3: heat 16384^2 fp32, 100 iterations (1 GPU)
timeout 600 python bench.py --config heat --steps 2 --no-cpu > $O/bench_heat.json 2> $O/bench_heat.err
# config 4: asymmetric (5,1,3,0) nearest, 4096^2 fp32, full wc x wr sweep, 30 samples
timeout 900 paper_1511_02490_b200/lib/wgtb collect --scenarios results/config4/descriptors --out $O/config4_samples.csv \
  --refused $O/config4_refused.csv --contexts $O/config4_contexts.csv --samples 30 --warmup 3 --store mean \
  > $O/config4.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:k_stencil_tma -s 2 -c 1 \
  -o $O/prof_boxmean5130_64x4 python scripts/profile_pass.py boxmean float32 4096 4096 64 4 4 auto nearest > /dev/null 2>&1
# race / memory checks of the smem-tile kernels (small grids: sanitizer is slow)
for args in "gol int32 auto 32 8 97 130" "boxmean float32 auto 16 6 70 90 nearest 0 5 1 3 0" "gaussian float64 explicit 8 8 50 64 pad 0.5 3 3 3 3" "heat float32 auto 6 10 61 77 nearest"; do
  timeout 300 compute-sanitizer --tool racecheck --racecheck-report hazard python scripts/probe_paths.py $args >> $O/sanitizer_racecheck.log 2>&1
  timeout 300 compute-sanitizer --tool memcheck python scripts/probe_paths.py $args >> $O/sanitizer_memcheck.log 2>&1
done
grep -E "RESULT|ERROR SUMMARY|hazard" $O/sanitizer_*.log | sort | uniq -c > $O/sanitizer_summary.txt
ls -la $O
