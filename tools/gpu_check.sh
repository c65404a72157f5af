#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_train.py tests/test_gpu_f2.py -x -q > gpurun_out/pytest_train.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_train.log
timeout 1500 python bench.py --dump-profile gpurun_out/profile_cfg2j.json > gpurun_out/bench_cfg2j.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_cfg2j.log
timeout 1500 python bench.py --fuse 1 --no-cpu > gpurun_out/bench_cfg2j_f2.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_cfg2j_f2.log
