#!/bin/bash
# The committed default line on the final code (+ smoke).
O=gpurun_out/r02z
mkdir -p $O
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench_cfg3.json 2> $O/bench_cfg3.err
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc $?" >> $O/smoke.log
timeout 900 python -m pytest tests/test_gpu_ops.py tests/test_gpu_train.py -q > $O/pytest_core.log 2>&1; echo "rc $?" >> $O/pytest_core.log
ls -la $O
