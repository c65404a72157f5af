#!/bin/bash
mkdir -p gpurun_out
POOCH_EARLY_AB=1 timeout 900 python -m pytest tests/test_gpu_ops.py -x -q -k "conv_fwd or dgrad" > gpurun_out/pytest_early.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_early.log
B=256 timeout 600 python tools/kbench_r50.py > gpurun_out/kb_r50_base.log 2>&1
POOCH_EARLY_AB=1 B=256 timeout 600 python tools/kbench_r50.py > gpurun_out/kb_r50_early.log 2>&1
timeout 1200 python bench.py --fuse 1 --no-cpu > gpurun_out/bench_cfg2_f2r.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_cfg2_f2r.log
