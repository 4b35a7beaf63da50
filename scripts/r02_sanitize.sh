#!/usr/bin/env bash
# compute-sanitizer on the round-2 kernels: the vector work-items and the NCCL
# halo schedule (thread-ranks over the NCCL test double).
cd "$(dirname "$0")/.."
O=gpurun_out/r02san; mkdir -p $O
for tool in memcheck racecheck initcheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_vector.py > $O/vector_$tool.log 2>&1
  echo "vector $tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' $O/vector_$tool.log | tail -1)"
done
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 paper_1511_02490_b200/lib/nccl_halo_test > $O/nccl_memcheck.log 2>&1
echo "nccl memcheck rc=$? $(grep -E 'ERROR SUMMARY' $O/nccl_memcheck.log | tail -1)"
