#!/usr/bin/env bash
# Warp-local edge fix-ups: parity (stencil, vector, fuzz, baseline configs, peer) then the landscape A/B.
cd "$(dirname "$0")/.."
O=gpurun_out/${1:-r04w}; mkdir -p $O
timeout 1500 python -m pytest tests/test_stencil_parity.py tests/test_vector_path.py tests/test_fuzz_paths.py \
  tests/test_baseline_configs.py tests/test_peer_halo.py tests/test_nccl_halo.py -m gpu -q -x > $O/pytest.log 2>&1
rc=$?; echo "pytest rc=$rc" | tee -a $O/pytest.log; tail -3 $O/pytest.log
if [ $rc = 0 ]; then
for r in 1 2; do
  SK_WARP_FIXUP=0 timeout 900 python scripts/landscape_probe.py 7 >> $O/land.jsonl 2>> $O/land.err
  timeout 900 python scripts/landscape_probe.py 7 >> $O/land.jsonl 2>> $O/land.err
done
fi
wc -l $O/land.jsonl
