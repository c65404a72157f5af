mkdir -p gpurun_out/sp
timeout 900 python -m pytest tests/test_gpu_epi2.py tests/test_gpu_ops.py -x -q 2>&1 | tail -5 > gpurun_out/sp/pytest.log
for v in 1 0 1 0; do echo "W2=$v"; POOCH_W2=$v OPS=fwd,dgrad timeout 300 python tools/kbench.py 2>&1 | grep layer; done > gpurun_out/sp/kb.log
