# ncu evidence for round 1 (run under gpurun)
set -x
mkdir -p gpurun_out
# launch list of the bench command (cold-cache, serialised)
ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --wc 32 --wr 32 --no-e2e --no-cpu > gpurun_out/bench_under_ncu.log 2>&1
# full captures of the top kernel at three block shapes
for shp in "32 32" "64 4" "128 8"; do
  set -- $shp
  ncu --set full --clock-control none --import-source on -k regex:k_stencil -s 2 -c 1 -o gpurun_out/prof_gol_${1}x${2} python scripts/profile_pass.py gol int32 8192 8192 $1 $2 4 > /dev/null 2>&1
done
ncu --set full --clock-control none --import-source on -k regex:k_stencil -s 2 -c 1 -o gpurun_out/prof_gol_explicit_32x8 python scripts/profile_pass.py gol int32 8192 8192 32 8 4 explicit > /dev/null 2>&1
ls -la gpurun_out
