#!/bin/bash
# The secondary workloads on the final code.
O=gpurun_out/r02ad
mkdir -p $O
timeout 900 python bench.py --workload alexnet --steps 10 --warmup 3 --no-cpu > $O/bench_alexnet.json 2> $O/bench_alexnet.err
timeout 900 python bench.py --workload cfg2 --ablation --steps 10 --warmup 3 --no-incore --no-cpu --no-check \
  > $O/bench_cfg2_ablation.json 2> $O/bench_cfg2_ablation.err
timeout 1200 python bench.py --workload resnext3d --steps 10 --warmup 3 > $O/bench_resnext3d.json 2> $O/bench_resnext3d.err
timeout 1500 python bench.py --workload cfg4 --steps 3 --warmup 3 --no-cpu --no-check --no-paper \
  > $O/bench_cfg4.json 2> $O/bench_cfg4.err
B=256 PREC=1 timeout 600 python tools/kbench_r50.py > $O/kbench_r50.log 2>&1
cp gpurun_out/kbench_r50_B256.json $O/kbench_r50_B256.json
ls -la $O
