#!/bin/bash
# W2 with three products (hi*[B;Bs] N=128 + lo*B N=64, default) vs four (lo*[B;Bs] + hi*[B;Bs], variant).
O=gpurun_out/r02r
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_ops.py tests/test_gpu_epi2.py -q -x > $O/pytest_ops.log 2>&1; echo "rc $?" >> $O/pytest_ops.log
for i in 1 2; do
  for v in three four; do
    L=""; [ $v = four ] && L="POOCH_LIB=paper_1907_05013_b200/libpooch_four.so"
    env $L B=256 PREC=1 timeout 600 python tools/kbench_r50.py > $O/kbench_${v}_$i.log 2>&1
    cp gpurun_out/kbench_r50_B256.json $O/kbench_${v}_$i.json
  done
done
ls -la $O
