#!/bin/bash
# Upper bound of halo reuse: A box loaded once per 9 k-blocks (POOCH_EPI_DIRECT=9, wrong results).
O=gpurun_out/r02n
mkdir -p $O
for v in 0 9 0 9; do
  POOCH_EPI_DIRECT=$v B=256 PREC=1 OPS=fwd,dgrad timeout 300 python tools/kbench.py > $O/kb_$v.log 2>&1
  cat $O/kb_$v.log >> $O/all.log
done
