#!/bin/bash
# Round-2 final measurements on the final code (three-product W2, wgrad split cap) -> gpurun_out/r02u/.
O=gpurun_out/r02u
mkdir -p $O
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench_cfg3.json 2> $O/bench_cfg3.err
for i in 2 3; do
  timeout 600 python bench.py --steps 20 --warmup 5 --no-incore --no-cpu --no-check --no-paper --no-cfg2 \
    > $O/bench_cfg3_run$i.json 2> $O/bench_cfg3_run$i.err
done
B=256 PREC=1 timeout 600 python tools/kbench_r50.py > $O/kbench_r50.log 2>&1
cp gpurun_out/kbench_r50_B256.json $O/kbench_r50_B256.json
timeout 900 python bench.py --workload alexnet --steps 10 --warmup 3 --no-cpu > $O/bench_alexnet.json 2> $O/bench_alexnet.err
timeout 900 python bench.py --workload cfg2 --ablation --steps 10 --warmup 3 --no-incore --no-cpu --no-check \
  > $O/bench_cfg2_ablation.json 2> $O/bench_cfg2_ablation.err
timeout 1200 python bench.py --workload resnext3d --steps 10 --warmup 3 > $O/bench_resnext3d.json 2> $O/bench_resnext3d.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --profile-from-start off --csv --log-file $O/launches_cfg3.csv \
  python bench.py --ncu-step --no-paper --no-cpu --no-incore --profile-repeats 1 > $O/ncu_step.log 2>&1
python tools/summarize_launches.py $O/launches_cfg3.csv $O/launches_summary_cfg3.txt \
  "ncu launch list of one cfg3 step (ResNet-50 batch 2560, all HBM), serialised, cold cache" > /dev/null
python tools/traffic_from_launches.py $O/launches_cfg3.csv $O/ncu_traffic.json cfg3 > /dev/null
rm -f $O/launches_cfg3.csv
timeout 2400 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc $?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc $?" >> $O/smoke.log
ls -la $O
