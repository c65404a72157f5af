#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ops.py -x -q -k "bnrelu or wgrad" > gpurun_out/pytest_f2ops.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_f2ops.log
timeout 900 python -m pytest tests/test_gpu_f2.py -x -q > gpurun_out/pytest_f2.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_f2.log
timeout 1200 python bench.py --fuse 1 --no-cpu --dump-profile gpurun_out/profile_cfg2_f2.json > gpurun_out/bench_cfg2_f2.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_cfg2_f2.log
