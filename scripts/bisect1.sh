set -x
P="python scripts/probe_paths.py"
for args in "gol int32 explicit 32 8 257 300" "gol int32 tma 32 8 257 300" "gol int32 tma 32 8 256 256" "five_point float32 tma 32 8 256 256" "five_point float64 tma 32 8 256 256" "five_point float32 tma 4 2 64 64"; do
  timeout 60 $P $args 2>&1 | grep -E "RESULT|Error|error|probe" | head -5
done
CUDA_LAUNCH_BLOCKING=1 timeout 120 compute-sanitizer --print-limit 5 python scripts/probe_paths.py gol int32 tma 32 8 256 256 2>&1 | head -40
cuobjdump -sass paper_1511_02490_b200/lib/libsk_stencil.so 2>/dev/null | grep -n "k_stencil_tma.*Gol.*int" | head -3
