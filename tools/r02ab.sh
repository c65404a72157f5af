#!/bin/bash
# Final code of the session: default line, GPU suite, smoke.
O=gpurun_out/r02ab
mkdir -p $O
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench_cfg3.json 2> $O/bench_cfg3.err
timeout 600 python bench.py --steps 20 --warmup 5 --no-incore --no-cpu --no-check --no-paper --no-cfg2 > $O/bench_cfg3_run2.json 2> $O/bench_cfg3_run2.err
timeout 2400 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc $?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc $?" >> $O/smoke.log
ls -la $O
