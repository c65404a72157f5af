#!/bin/bash
# BN kernels: evict-first (streaming) feature-map loads / stores (default) vs plain (variant), in-core ResNet-50 b640.
O=gpurun_out/r02w
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_ops.py -q -x -k "bn or BN" > $O/pytest_bn.log 2>&1; echo "rc $?" >> $O/pytest_bn.log
for i in 1 2; do
  for v in stream plain; do
    L=""; [ $v = plain ] && L="POOCH_LIB=paper_1907_05013_b200/libpooch_nostream.so"
    env $L timeout 600 python bench.py --workload cfg2 --budget-gib 170 --steps 10 --warmup 3 --no-incore --no-cpu \
      --no-check --no-paper --no-cfg2 > $O/incore_${v}_$i.json 2> $O/incore_${v}_$i.err
  done
done
ls -la $O
