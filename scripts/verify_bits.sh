#!/usr/bin/env bash
cd "$(dirname "$0")/.."
O=gpurun_out/bits1; mkdir -p $O
timeout 900 python -m pytest tests/test_gol_bits.py -q -x > $O/pytest_bits.log 2>&1; echo "rc=$?" >> $O/pytest_bits.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 tests/mp_gpu_worker.py > $O/mp.log 2>&1
timeout 1200 python scripts/bits_probe.py > $O/bits_probe.txt 2>&1
tail -5 $O/pytest_bits.log; tail -3 $O/mp.log; tail -45 $O/bits_probe.txt
