#!/bin/bash
# On the GPU box: GPU tests, per-shape conv microbench, the default bench line (profile dumped).
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
B=256 timeout 600 python tools/kbench_r50.py > gpurun_out/kb_r50.log 2>&1
timeout 1200 python bench.py --dump-profile gpurun_out/profile_cfg2f.json > gpurun_out/bench_cfg2f.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_cfg2f.log
