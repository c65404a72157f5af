mkdir -p gpurun_out
for m in 0 1; do
  if [ $m = 1 ]; then export POOCH_EXP_BULK_B=1; fi
  B=256 ONLY="l1.c2" OPS=fwd,dgrad timeout 300 python tools/kbench.py > gpurun_out/expb_l1c2_$m.log 2>&1
  B=256 ONLY="l3.c2" OPS=fwd,dgrad timeout 300 python tools/kbench.py > gpurun_out/expb_l3c2_$m.log 2>&1
  B=256 ONLY="l1.c1" OPS=fwd,dgrad timeout 300 python tools/kbench.py > gpurun_out/expb_l1c1_$m.log 2>&1
done
