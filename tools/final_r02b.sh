#!/bin/bash
# Round-2 re-measurement with the final kernels (transpose-free wgrad, grouped conv v3) on one
# B200; outputs under gpurun_out/r02h/.
O=gpurun_out/r02h
mkdir -p $O
for i in 2 3; do
  timeout 600 python bench.py --steps 20 --warmup 5 --no-incore --no-cpu --no-check --no-paper --no-cfg2 \
    > $O/bench_cfg3_run$i.json 2> $O/bench_cfg3_run$i.err
done
timeout 900 python bench.py --workload alexnet --steps 10 --warmup 3 --no-cpu > $O/bench_alexnet.json 2> $O/bench_alexnet.err
timeout 900 python bench.py --workload cfg2 --ablation --steps 10 --warmup 3 --no-incore --no-cpu --no-check \
  > $O/bench_cfg2_ablation.json 2> $O/bench_cfg2_ablation.err
timeout 1200 python bench.py --workload cfg4 --steps 3 --warmup 3 --no-cpu --no-check --no-paper \
  > $O/bench_cfg4.json 2> $O/bench_cfg4.err
ls -la $O
