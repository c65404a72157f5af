#!/bin/bash
# On the GPU box: cfg3 / cfg4 bench lines, then the cfg2 ncu launch list + full captures.
mkdir -p gpurun_out
bash tools/bench_all.sh
bash tools/ncu_run.sh > gpurun_out/ncu_run.log 2>&1
