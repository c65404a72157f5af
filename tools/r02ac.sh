#!/bin/bash
# Full ncu captures of the dominant family's kernels on the final code (batch 256).
O=gpurun_out/r02ac
mkdir -p $O
bash tools/ncu_kernels.sh "l3.c2 3x3:wgrad" "l2.c2 3x3:wgrad" "l1.c2 3x3:wgrad" "l1.c2 3x3:dgrad" "stem7x7:wgrad"
for t in l3_c2_3x3-wgrad l2_c2_3x3-wgrad l1_c2_3x3-wgrad l1_c2_3x3-dgrad stem7x7-wgrad; do
  python tools/ncu_summarize_full.py gpurun_out/ncu/${t}_raw.csv "$t batch 256" >> $O/ncu_kernels.txt 2>&1
done
ls -la $O
