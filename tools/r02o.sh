#!/bin/bash
# Decoupled TMEM A-slot ring (TSPLIT): parity + kernel bench.
O=gpurun_out/r02o
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_ops.py tests/test_gpu_wgrad_mn.py tests/test_gpu_epi2.py -q -x > $O/pytest_ops.log 2>&1; echo "rc $?" >> $O/pytest_ops.log
for i in 1 2; do
B=256 PREC=1 timeout 600 python tools/kbench_r50.py > $O/kbench_$i.log 2>&1
cp gpurun_out/kbench_r50_B256.json $O/kbench_$i.json
done
ls -la $O
