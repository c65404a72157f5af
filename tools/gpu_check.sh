#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_ops.py -x -q > gpurun_out/pytest_ops.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_ops.log
B=256 timeout 600 python tools/kbench_r50.py > gpurun_out/kb_r50_at.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 1500 python bench.py --dump-profile gpurun_out/profile_cfg2n.json > gpurun_out/bench_cfg2n.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_cfg2n.log
