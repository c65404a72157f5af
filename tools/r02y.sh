#!/bin/bash
# wgrad split cap 2048: kernel bench at batch 256, cfg3 line, long-split accuracy.
O=gpurun_out/r02y
mkdir -p $O
B=256 PREC=1 timeout 600 python tools/kbench_r50.py > $O/kbench_r50.log 2>&1
cp gpurun_out/kbench_r50_B256.json $O/kbench_r50_B256.json
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-cfg2 --no-check --no-paper > $O/bench_cfg3.json 2> $O/bench_cfg3.err
timeout 1200 python tools/acc_split_probe.py > $O/acc_split_probe.log 2>&1
ls -la $O
