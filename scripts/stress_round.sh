set -x
O=gpurun_out/r01
rm -f $O/stress.log
for cfg in "heat float32 2048 2048 2 32 4000" "heat float32 2048 2048 2 16 3000" "heat float32 2048 2048 4 32 3000" "heat float32 4096 4096 2 32 1000" "five_point float32 2048 2048 2 32 3000 nearest 2" "gol int32 2048 2048 2 32 3000 pad 2" "heat float64 2048 2048 2 32 2000 nearest 2" "heat float32 2048 2048 2 32 2000 nearest 4" "heat float32 2048 2048 8 8 2000 nearest 8"; do
  timeout 600 python scripts/stress_race.py $cfg >> $O/stress.log 2>&1
done
grep RESULT $O/stress.log
