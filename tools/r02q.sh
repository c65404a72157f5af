#!/bin/bash
# BN backward apply: two elements per iteration (default) vs one (variant), in-core ResNet-50 b640.
O=gpurun_out/r02q
mkdir -p $O
for i in 1 2; do
  for v in new ilp1; do
    L=""; [ $v = ilp1 ] && L="POOCH_LIB=paper_1907_05013_b200/libpooch_ilp1.so"
    env $L timeout 600 python bench.py --workload cfg2 --budget-gib 170 --steps 10 --warmup 3 --no-incore --no-cpu \
      --no-check --no-paper --no-cfg2 > $O/incore_${v}_$i.json 2> $O/incore_${v}_$i.err
  done
done
ls -la $O
