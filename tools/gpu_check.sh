mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
B=256 timeout 600 python tools/kbench_r50.py > gpurun_out/kb_r50_staged.log 2>&1
cp gpurun_out/kbench_r50_B256.json gpurun_out/kbench_r50_B256_staged.json
POOCH_EPI_DIRECT=1 B=256 timeout 600 python tools/kbench_r50.py > gpurun_out/kb_r50_direct.log 2>&1
cp gpurun_out/kbench_r50_B256.json gpurun_out/kbench_r50_B256_direct.json
timeout 900 python bench.py --dump-profile gpurun_out/profile_cfg2b.json > gpurun_out/bench_cfg2b.log 2>&1
