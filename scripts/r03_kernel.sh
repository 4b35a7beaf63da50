#!/usr/bin/env bash
# Kernel change check: vector/box parity tests, the config-4 probe, the bench line.
cd "$(dirname "$0")/.."
O=gpurun_out/${1:-r03k}; mkdir -p $O
timeout 900 python -m pytest tests/test_vector_path.py tests/test_div_const.py tests/test_baseline_configs.py \
  "tests/test_stencil_parity.py::test_boxmean_division_special_values" -q -m gpu > $O/pytest.log 2>&1
echo "pytest rc=$?" | tee -a $O/pytest.log; tail -4 $O/pytest.log
timeout 600 python scripts/box_probe.py 30 > $O/box_probe.json 2> $O/box_probe.err; echo "probe rc=$?"
timeout 1200 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
tail -c 600 $O/bench.err
