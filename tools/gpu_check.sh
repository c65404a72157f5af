#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_ops.py -x -q > gpurun_out/pytest_ops.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_ops.log
B=256 timeout 600 python tools/kbench_r50.py > gpurun_out/kb_r50_naux.log 2>&1
