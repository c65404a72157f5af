#!/bin/bash
# wgrad split cap (1024 k-blocks): accuracy of long splits, cfg3 A/B.
O=gpurun_out/r02t
mkdir -p $O
timeout 1200 python tools/acc_split_probe.py > $O/acc_split_probe.log 2>&1
timeout 600 python -m pytest tests/test_gpu_ops.py -q -x -k wgrad > $O/pytest_wgrad.log 2>&1; echo "rc $?" >> $O/pytest_wgrad.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-cfg2 --no-check --no-paper > $O/bench_cap_1.json 2> $O/bench_cap_1.err
POOCH_WGRAD_KMAX=0 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-cfg2 --no-check --no-paper > $O/bench_nocap.json 2> $O/bench_nocap.err
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-cfg2 --no-check --no-paper > $O/bench_cap_2.json 2> $O/bench_cap_2.err
ls -la $O
