#!/usr/bin/env bash
cd "$(dirname "$0")/.."
O=gpurun_out/c10; mkdir -p $O
timeout 900 python -m pytest tests/test_stencil_parity.py tests/test_gol_bits.py -x -q -k "gol or Gol" > $O/pytest_gol.log 2>&1; echo "rc=$?" >> $O/pytest_gol.log
tail -3 $O/pytest_gol.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_stencil -s 2 -c 1 -o $O/prof_gol_144x4 python scripts/profile_pass.py gol int32 8192 8192 144 4 4 > $O/ncu.log 2>&1
tail -1 $O/ncu.log
timeout 900 python bench.py > $O/bench_gol.json 2> $O/bench_gol.err; echo "bench rc=$?"
cat $O/bench_gol.json
