#!/bin/bash
# Round-2 re-entry check: GPU suite, smoke, default bench line, kernel bench at batch 256.
O=gpurun_out/r02k
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc $?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc $?" >> $O/smoke.log
B=256 PREC=1 timeout 600 python tools/kbench_r50.py > $O/kbench.log 2>&1
cp gpurun_out/kbench_r50_B256.json $O/ 2>/dev/null
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err
ls -la $O
