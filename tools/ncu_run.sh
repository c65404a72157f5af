#!/bin/bash
# On the GPU box: launch list of one bench step + full captures of the dominant kernels.
B=${BATCH:-640}
mkdir -p gpurun_out
timeout 1200 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --ncu-step --batch $B --profile-iters 1 > gpurun_out/ncu_launch.log 2>&1
echo "launch list rc=$?"
timeout 1200 ncu --profile-from-start off --set full --clock-control none --import-source on \
  -k regex:igemm_kernel -c 4 -o gpurun_out/prof_igemm_step \
  python bench.py --ncu-step --batch $B --profile-iters 1 > gpurun_out/ncu_full.log 2>&1
echo "full igemm rc=$?"
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on \
  -k regex:"bn_bwd_apply|bn_apply" -c 2 -o gpurun_out/prof_bn_step \
  python bench.py --ncu-step --batch $B --profile-iters 1 > gpurun_out/ncu_full_bn.log 2>&1
echo "full bn rc=$?"
ls -la gpurun_out | tail
