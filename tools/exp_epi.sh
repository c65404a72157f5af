mkdir -p gpurun_out
for m in 0 2 3 4; do POOCH_EPI_DIRECT=$m B=256 ONLY="l1.c3" OPS=fwd timeout 300 python tools/kbench.py > gpurun_out/exp_epi$m.log 2>&1; done
for m in 0 2 3 4; do POOCH_EPI_DIRECT=$m B=256 ONLY="l3.c3" OPS=fwd timeout 300 python tools/kbench.py > gpurun_out/exp4_epi$m.log 2>&1; done
