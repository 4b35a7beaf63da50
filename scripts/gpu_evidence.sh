#!/usr/bin/env bash
# Round evidence on one B200 (run under gpurun): the GPU test suite, smoke,
# bench lines (headline GoL + config 3 heat + the reference arm), the launch
# list of the bench command, ncu --set full captures of the dominant kernels
# (one-pass GoL, register-strip heat, bit-plane strips), and sanitizer runs
# of the temporal paths.  Outputs land in gpurun_out/evidence/.
cd "$(dirname "$0")/.."
O=gpurun_out/evidence; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" | tee -a $O/pytest_gpu.log
tail -2 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > $O/bench_gol.json 2> $O/bench_gol.err; echo "bench rc=$?"
timeout 900 python bench.py --config heat --steps 10 > $O/bench_heat.json 2> $O/bench_heat.err; echo "bench heat rc=$?"
timeout 900 python bench.py --impl reference --steps 3 > $O/bench_reference.json 2> $O/bench_reference.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/launches_gol_bench.csv \
  python bench.py --steps 2 --warmup 3 --wc 128 --wr 8 --no-e2e --no-cpu --no-temporal > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_stencil_tma -s 2 -c 1 \
  -o $O/prof_gol_128x8 python scripts/profile_pass.py gol int32 8192 8192 128 8 4 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_cross_strips -s 1 -c 1 \
  -o $O/prof_strips_heat python scripts/profile_strips.py 16384 8 8 32 12 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gol_strips -s 1 -c 1 \
  -o $O/prof_bits python scripts/profile_bits.py 8192 10 32 12 16 1 > /dev/null 2>&1
for k in strips bitplane fused peer streamed; do
  timeout 300 compute-sanitizer --tool racecheck --racecheck-report hazard python scripts/sanitize_temporal.py $k >> $O/sanitizer_racecheck.log 2>&1
  timeout 300 compute-sanitizer --tool memcheck python scripts/sanitize_temporal.py $k >> $O/sanitizer_memcheck.log 2>&1
done
grep -E "ERROR SUMMARY|RACECHECK SUMMARY" $O/sanitizer_*.log | sort | uniq -c
# digests + raw pages stay; the .ncu-rep files would exceed gpurun's 64 MiB copy-back
for p in prof_gol_128x8 prof_strips_heat prof_bits; do
  python scripts/ncu_digest.py $O/$p.ncu-rep > $O/${p}_digest.txt 2>/dev/null
  ncu -i $O/$p.ncu-rep --page raw --csv > $O/${p}_raw.csv 2>/dev/null
  [ -s $O/${p}_digest.txt ] && rm -f $O/$p.ncu-rep
done
ls -la $O
