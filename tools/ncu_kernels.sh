#!/bin/bash
# Full ncu captures (source-correlated) of single conv passes on ResNet-50 shapes (batch 256).
# Usage on the GPU box: bash tools/ncu_kernels.sh "l1.c3 1x1:fwd" "l1.c2 3x3:wgrad" ...
mkdir -p gpurun_out/ncu
for spec in "$@"; do
  only="${spec%%:*}"; op="${spec##*:}"; tag=$(echo "$only-$op" | tr ' .' '__')
  ONLY="$only" OPS="$op" B=256 timeout 600 ncu --set full --import-source on --clock-control none \
    -k regex:igemm --launch-skip 2 -c 1 -f -o gpurun_out/ncu/$tag python tools/kbench.py > gpurun_out/ncu/$tag.log 2>&1
  ncu -i gpurun_out/ncu/$tag.ncu-rep --page raw --csv > gpurun_out/ncu/${tag}_raw.csv 2>/dev/null
  ncu -i gpurun_out/ncu/$tag.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu/${tag}_sass.csv 2>/dev/null
  gzip -f gpurun_out/ncu/${tag}_sass.csv
  rm -f gpurun_out/ncu/$tag.ncu-rep
done
