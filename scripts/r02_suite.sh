#!/usr/bin/env bash
# Full GPU suite (no -x: every failure listed) + the driver's smoke().
cd "$(dirname "$0")/.."
O=gpurun_out/${1:-r02c}; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" | tee -a $O/pytest_gpu.log
tail -15 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" | tee -a $O/smoke.log
