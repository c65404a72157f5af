mkdir -p gpurun_out/sp
for d in 0 7 8 0; do echo "EPI_DIRECT=$d"; POOCH_EPI_DIRECT=$d ONLY=stem OPS=fwd timeout 300 python tools/kbench.py 2>&1 | grep layer; done > gpurun_out/sp/abl.log
for d in 0 8; do echo "RELAY EPI_DIRECT=$d"; POOCH_LIB=paper_1907_05013_b200/libpooch_relay.so POOCH_EPI_DIRECT=$d ONLY=stem OPS=fwd timeout 300 python tools/kbench.py 2>&1 | grep layer; done >> gpurun_out/sp/abl.log
timeout 600 python -m pytest tests/test_gpu_epi2.py -x -q -k stem 2>&1 | tail -2 >> gpurun_out/sp/abl.log
