#!/bin/bash
# Round-2 measurement session on one B200 (outputs under gpurun_out/r02f/).
set -x
O=gpurun_out/r02f
mkdir -p $O
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench_cfg3.json 2> $O/bench_cfg3.err
for i in 2 3; do
  timeout 600 python bench.py --steps 20 --warmup 5 --no-incore --no-cpu --no-check --no-paper \
    > $O/bench_cfg3_run$i.json 2> $O/bench_cfg3_run$i.err
done
timeout 900 python bench.py --workload cfg2 --ablation --steps 10 --warmup 3 --no-incore --no-cpu --no-check \
  > $O/bench_cfg2_ablation.json 2> $O/bench_cfg2_ablation.err
timeout 900 python bench.py --workload cfg4 --steps 3 --warmup 3 --no-cpu --no-check --no-paper \
  > $O/bench_cfg4.json 2> $O/bench_cfg4.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --profile-from-start off --csv --log-file $O/launches_cfg3.csv \
  python bench.py --ncu-step --no-paper --no-cpu --no-incore --profile-repeats 1 > $O/ncu_step.log 2>&1
python tools/summarize_launches.py $O/launches_cfg3.csv $O/launches_summary_cfg3.txt \
  "ncu launch list of one cfg3 step (ResNet-50 batch 2560, all HBM), serialised, cold cache" > /dev/null
python tools/traffic_from_launches.py $O/launches_cfg3.csv $O/ncu_traffic.json > /dev/null
ls -la $O
