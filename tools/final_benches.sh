#!/bin/bash
# On the GPU box: cfg3 / cfg4 bench lines on the final code.
mkdir -p gpurun_out
bash tools/bench_all.sh
