mkdir -p gpurun_out/e2
python -m pytest tests/test_gpu_epi2.py -x -q 2>&1 | tail -5 | tee gpurun_out/e2/pytest.log
for d in 0 5 0 5; do echo "EPI_DIRECT=$d"; POOCH_EPI_DIRECT=$d OPS=fwd,dgrad timeout 300 python tools/kbench.py 2>&1 | grep layer; done > gpurun_out/e2/batched.log
