#!/usr/bin/env bash
cd "$(dirname "$0")/.."
O=gpurun_out/c13; mkdir -p $O
timeout 900 python -m pytest tests/test_cpp_api.py tests/test_stencil_parity.py -x -q -k "cpp or streamed or api" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
tail -3 $O/pytest.log
timeout 900 python bench.py > $O/bench_gol.json 2> $O/bench_gol.err; echo "bench rc=$?"
cat $O/bench_gol.json
timeout 900 python bench.py --impl reference --steps 3 > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref rc=$?"
cat $O/bench_ref.json
