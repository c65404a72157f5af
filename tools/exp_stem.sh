mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_ops.py -x -q -k "conv_fwd" > gpurun_out/pytest_stem.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_stem.log
timeout 600 python -m pytest tests/test_gpu_train.py -x -q -k tiny > gpurun_out/pytest_tiny.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_tiny.log
for p in 0 1; do PREC=$p B=256 ONLY=stem OPS=fwd timeout 300 python tools/kbench.py > gpurun_out/exps_$p.log 2>&1; done
