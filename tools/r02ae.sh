#!/bin/bash
# Two more default-line runs on the final code (run-to-run spread).
O=gpurun_out/r02ae
mkdir -p $O
for i in 3 4; do
  timeout 600 python bench.py --steps 20 --warmup 5 --no-incore --no-cpu --no-check --no-paper --no-cfg2 \
    > $O/bench_cfg3_run$i.json 2> $O/bench_cfg3_run$i.err
done
ls -la $O
