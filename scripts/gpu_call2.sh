#!/usr/bin/env bash
# pytest -m gpu, bit-plane ncu evidence (full capture of k_gol_strips + launch
# list of one 100-generation run), heat temporal-blocking probe.
cd "$(dirname "$0")/.."
O=gpurun_out/c2; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
tail -3 $O/pytest_gpu.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gol_strips -s 1 -c 1 \
  -o $O/prof_bits_tb10_32x12_k16 python scripts/profile_bits.py 8192 10 32 12 16 1 > $O/ncu_full.log 2>&1
tail -2 $O/ncu_full.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file $O/launches_bits.csv python scripts/profile_bits.py 8192 10 32 12 16 1 > $O/ncu_list.log 2>&1
tail -2 $O/ncu_list.log
timeout 900 python scripts/tb_probe.py heat float32 16384 100 > $O/tb_heat.txt 2>&1
cat $O/tb_heat.txt | head -20
