#!/bin/bash
# ResNeXt-101 (3D) open item: do identical launches slow down with the budget (arena fullness)?
O=gpurun_out/r02x
mkdir -p $O
for b in 16 24 40; do
  timeout 900 python bench.py --workload resnext3d --budget-gib $b --steps 10 --warmup 3 --no-cpu --no-check --no-paper \
    > $O/rx_$b.json 2> $O/rx_$b.err
done
ls -la $O
