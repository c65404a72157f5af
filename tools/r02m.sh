#!/bin/bash
# Stem patch wgrad (SPW) + W2 wgrad: parity, then kernel bench A/B at batch 256.
O=gpurun_out/r02m
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_ops.py tests/test_gpu_wgrad_mn.py -q -x > $O/pytest_ops.log 2>&1; echo "rc $?" >> $O/pytest_ops.log
for v in default w2off spwoff; do
  case $v in
    default) E="";;
    w2off) E="POOCH_WGRAD_W2=0";;
    spwoff) E="POOCH_STEM_PATCH_WGRAD=0";;
  esac
  env $E B=256 PREC=1 timeout 600 python tools/kbench_r50.py > $O/kbench_$v.log 2>&1
  cp gpurun_out/kbench_r50_B256.json $O/kbench_$v.json
done
ls -la $O
