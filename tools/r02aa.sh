#!/bin/bash
# W2 with hi read from the smem stage (lo only into TMEM, default) vs hi + lo in TMEM (variant).
O=gpurun_out/r02aa
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_ops.py tests/test_gpu_epi2.py tests/test_gpu_f2.py -q -x > $O/pytest.log 2>&1; echo "rc $?" >> $O/pytest.log
for i in 1 2; do
  for v in hismem hitmem; do
    L=""; [ $v = hitmem ] && L="POOCH_LIB=paper_1907_05013_b200/libpooch_hitmem.so"
    env $L B=256 PREC=1 timeout 600 python tools/kbench_r50.py > $O/kbench_${v}_$i.log 2>&1
    cp gpurun_out/kbench_r50_B256.json $O/kbench_${v}_$i.json
  done
done
ls -la $O
