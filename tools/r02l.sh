#!/bin/bash
# Shared-link model A/B on cfg3 + GPU suite.
O=gpurun_out/r02l
mkdir -p $O
for i in 1 2; do
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-cfg2 --no-check > $O/bench_cfg3_duplex_$i.json 2> $O/bench_cfg3_duplex_$i.err
done
POOCH_DUPLEX=0 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-cfg2 --no-check --no-incore --no-paper > $O/bench_cfg3_noduplex.json 2> $O/bench_cfg3_noduplex.err
timeout 2400 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc $?" >> $O/pytest_gpu.log
ls -la $O
