#!/bin/bash
# On the GPU box: the full GPU test suite, smoke(), and the default bench line.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
timeout 1500 python bench.py --dump-profile gpurun_out/profile_cfg2_final.json > gpurun_out/bench_cfg2_final.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_cfg2_final.log
