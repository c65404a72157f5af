#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 1500 python bench.py --dump-profile gpurun_out/profile_cfg2k.json > gpurun_out/bench_cfg2k.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_cfg2k.log
