#!/bin/bash
# On the GPU box: launch list of one bench step (cfg2 by default) + full captures of the
# dominant kernels (TMA conv fwd / dgrad / wgrad, BN). Output under gpurun_out/.
B=${BATCH:-640}
mkdir -p gpurun_out
timeout 1200 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --ncu-step --batch $B --profile-iters 1 > gpurun_out/ncu_launch.log 2>&1
echo "launch list rc=$?"
# skip the stem (cp.async path) and take a spread of TMA forward convs
timeout 1500 ncu --profile-from-start off --set full --clock-control none --import-source on \
  --kernel-name-base demangled -k regex:"igemm_kernel<\\(int\\)0" -s 1 -c 6 -o gpurun_out/prof_fwd_step \
  python bench.py --ncu-step --batch $B --profile-iters 1 > gpurun_out/ncu_full_fwd.log 2>&1
echo "full fwd rc=$?"
timeout 1200 ncu --profile-from-start off --set full --clock-control none --import-source on \
  --kernel-name-base demangled -k regex:"igemm_kernel<\\(int\\)[12]" -c 6 -o gpurun_out/prof_bwd_step \
  python bench.py --ncu-step --batch $B --profile-iters 1 > gpurun_out/ncu_full_bwd.log 2>&1
echo "full bwd rc=$?"
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on \
  -k regex:"bn_bwd_apply|bn_apply|maxpool" -c 4 -o gpurun_out/prof_bn_step \
  python bench.py --ncu-step --batch $B --profile-iters 1 > gpurun_out/ncu_full_bn.log 2>&1
echo "full bn rc=$?"
ls -la gpurun_out | tail
