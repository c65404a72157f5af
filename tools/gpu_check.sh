#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_ops.py -x -q -k bnrelu > gpurun_out/pytest_f2ops.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_f2ops.log
timeout 900 python -m pytest tests/test_gpu_f2.py -x -q > gpurun_out/pytest_f2.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_f2.log
timeout 1500 python bench.py --fuse 1 --no-cpu > gpurun_out/bench_f2x.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_f2x.log
timeout 1500 python bench.py --no-cpu > gpurun_out/bench_plainx.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_plainx.log
