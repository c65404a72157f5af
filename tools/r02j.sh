O=gpurun_out/r02j
mkdir -p $O
timeout 600 python tools/kbench_r50.py > $O/kbench_r50.log 2>&1
cp gpurun_out/kbench_r50_B256.json $O/ 2>/dev/null
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench_cfg3.json 2> $O/bench_cfg3.err
