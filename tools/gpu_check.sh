#!/bin/bash
# On the GPU box: GPU tests (f2 first), then the default bench line plain and with f2 fusion.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ops.py -x -q -k bnrelu > gpurun_out/pytest_f2ops.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_f2ops.log
timeout 900 python -m pytest tests/test_gpu_f2.py -x -q > gpurun_out/pytest_f2.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_f2.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 1200 python bench.py --fuse 1 --no-cpu --dump-profile gpurun_out/profile_cfg2_f2.json > gpurun_out/bench_cfg2_f2.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_cfg2_f2.log
