#!/bin/bash
# On the GPU box: launch list of one cfg2 bench step (every kernel: duration + DRAM bytes) and
# ncu --set full captures of the dominant kernels (TMA conv fwd / dgrad / wgrad, BN, pool),
# exported as raw CSV (the .ncu-rep files stay on the box: gpurun_out is capped at 64 MiB).
B=${BATCH:-640}
mkdir -p gpurun_out
timeout 1200 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --ncu-step --batch $B --profile-iters 1 > gpurun_out/ncu_launch.log 2>&1
echo "launch list rc=$?"
full() {  # name, kernel regex, launch-skip, count
  timeout 1500 ncu --profile-from-start off --set full --clock-control none --import-source on \
    --kernel-name-base demangled -k regex:"$2" -s $3 -c $4 -o /tmp/$1 \
    python bench.py --ncu-step --batch $B --profile-iters 1 > gpurun_out/ncu_$1.log 2>&1
  echo "$1 rc=$?"
  ncu -i /tmp/$1.ncu-rep --page raw --csv > gpurun_out/$1_raw.csv 2>/dev/null
  gzip -f gpurun_out/$1_raw.csv
}
full prof_fwd_step 'igemm_kernel<\(int\)0' 1 6
full prof_bwd_step 'igemm_kernel<\(int\)[12]' 2 6
full prof_bn_step 'bn_bwd_apply|bn_apply|maxpool' 0 4
ls -la gpurun_out
