#!/bin/bash
# On the GPU box: the other BASELINE configs' bench lines (cfg3: ResNet-50 b2560 in all HBM;
# cfg4: 3D U-Net 256^3), W=3 warm-up steps.
mkdir -p gpurun_out
timeout 1500 python bench.py --workload cfg3 --steps 3 --warmup 3 --no-cpu --dump-profile gpurun_out/profile_cfg3.json > gpurun_out/bench_cfg3.log 2>&1; echo "cfg3 rc=$?" >> gpurun_out/bench_cfg3.log
timeout 1500 python bench.py --workload cfg4 --steps 2 --warmup 3 --no-cpu > gpurun_out/bench_cfg4.log 2>&1; echo "cfg4 rc=$?" >> gpurun_out/bench_cfg4.log
