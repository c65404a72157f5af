#!/bin/bash
mkdir -p gpurun_out
timeout 2400 python bench.py --ablation --no-cpu > gpurun_out/bench_ablation.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_ablation.log
