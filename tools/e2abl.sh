mkdir -p gpurun_out/e2
for d in 0 3 4 2 0; do echo "EPI_DIRECT=$d"; POOCH_EPI_DIRECT=$d ONLY=l1.c3 OPS=fwd,dgrad timeout 300 python tools/kbench.py 2>&1 | grep layer; done > gpurun_out/e2/abl.log
for d in 0 3 4 2; do echo "EPI2=0 EPI_DIRECT=$d"; POOCH_EPI2=0 POOCH_EPI_DIRECT=$d ONLY=l1.c3 OPS=fwd timeout 300 python tools/kbench.py 2>&1 | grep layer; done >> gpurun_out/e2/abl.log
