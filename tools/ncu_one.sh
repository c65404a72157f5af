#!/bin/bash
# On the GPU box: ncu --set full of ONE conv launch of tools/kbench.py (ONLY=<layer> OPS=<op>),
# exported as raw metrics + per-source-line (SASS) CSV.
mkdir -p gpurun_out
tag=${TAG:-one}
B=${B:-256} ONLY=$ONLY OPS=$OPS timeout 900 ncu --set full --clock-control none --import-source on \
  --kernel-name-base demangled -k regex:igemm -s 2 -c 1 -o /tmp/$tag python tools/kbench.py > gpurun_out/ncu_$tag.log 2>&1
ncu -i /tmp/$tag.ncu-rep --page raw --csv > gpurun_out/${tag}_raw.csv 2>/dev/null
ncu -i /tmp/$tag.ncu-rep --page source --csv --print-source sass > gpurun_out/${tag}_sass.csv 2>/dev/null
ncu -i /tmp/$tag.ncu-rep --page details --csv > gpurun_out/${tag}_details.csv 2>/dev/null
gzip -f gpurun_out/${tag}_*.csv
