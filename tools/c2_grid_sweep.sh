#!/bin/bash
# C2 (N=1) put grid-shape sweep: payload GB/s of the default bench line per
# (ctas, threads) pair, each run twice.  Output: gpurun_out/c2_grid_sweep.txt
out=gpurun_out/c2_grid_sweep.txt
echo "# ctas threads value_GBps put_avg_ms (bench.py N=1 C2, default steps)" > $out
for cfg in "0 256" "0 224" "0 288" "148 224" "296 128" "296 96" "0 256" "0 224"; do
  set -- $cfg
  line=$(timeout 200 python bench.py --ctas $1 --threads $2 2>/dev/null | tail -1)
  v=$(python -c "import json,sys; d=json.loads(sys.argv[1]); print(d['value'], d['kernels_ms']['put_avg'], d['roofline']['frac'])" "$line" 2>/dev/null)
  echo "$1 $2 $v" >> $out
done
