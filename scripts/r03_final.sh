#!/usr/bin/env bash
# Full GPU suite + smoke + bench on the current build; then, if the suite
# passed, the real-kernel re-sweep (scripts/r03_resweep.sh) on this executor.
cd "$(dirname "$0")/.."
O=gpurun_out/${1:-r03f}; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; rc=$?
echo "pytest rc=$rc" | tee -a $O/pytest_gpu.log; tail -6 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" | tee -a $O/smoke.log
timeout 600 python scripts/box_probe.py 30 > $O/box_probe.json 2> $O/box_probe.err; echo "probe rc=$?"
timeout 1200 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
if [ $rc = 0 ] && [ "${SWEEP:-1}" = 1 ]; then
  SWEEP_SECONDS=${SWEEP_SECONDS:-4200} bash scripts/r03_resweep.sh > $O/resweep.log 2>&1; echo "resweep rc=$?"
fi
