#!/bin/bash
# Run on the GPU box (gpurun): launch list of one bench step + a full ncu capture of the
# dominant kernel. Outputs land in gpurun_out/ (merged back), summarised into profiles/.
set -x
B=${BATCH:-640}
mkdir -p gpurun_out
# 1) launch list of the timed region of a short bench run (cold-cache, serialised)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches.csv \
  python bench.py --steps 1 --warmup 1 --no-incore --no-cpu --batch $B > gpurun_out/ncu_bench.log 2>&1
# 2) full capture of the top kernels (a few launches each)
timeout 1200 ncu --set full --clock-control none --import-source on \
  -k regex:igemm_kernel -s 200 -c 6 -o gpurun_out/prof_igemm \
  python bench.py --steps 1 --warmup 0 --no-incore --no-cpu --batch $B > gpurun_out/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"bn_bwd|bn_apply" -s 100 -c 4 -o gpurun_out/prof_bn \
  python bench.py --steps 1 --warmup 0 --no-incore --no-cpu --batch $B > gpurun_out/ncu_full_bn.log 2>&1
ls -la gpurun_out
