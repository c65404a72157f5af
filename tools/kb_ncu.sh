#!/bin/bash
# On the GPU box: conv-op parity tests, per-layer kernel microbench (B=256) and ncu --set full
# of every conv launch of the microbench, exported as raw CSV (the .ncu-rep stays on the box).
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_ops.py -x -q > gpurun_out/pytest_ops.log 2>&1; echo "ops rc=$?"
B=256 timeout 600 python tools/kbench.py > gpurun_out/kbench_all.log 2>&1; echo "kbench rc=$?"
B=256 OPS=${OPS:-fwd} timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k regex:igemm -c ${NCU_C:-80} -o /tmp/prof_kb python tools/kbench.py > gpurun_out/ncu_kb.log 2>&1
echo "ncu rc=$?"
ncu -i /tmp/prof_kb.ncu-rep --page raw --csv > gpurun_out/ncu_kb_raw.csv 2>/dev/null
gzip -f gpurun_out/ncu_kb_raw.csv
ls -la gpurun_out
