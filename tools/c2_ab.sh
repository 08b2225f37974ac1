#!/bin/bash
# Same-box A/B of the C2 bench line: library default (224 threads) vs 256 threads, alternating.
out=gpurun_out/c2_ab.txt
echo "# threads value_GBps put_avg_ms roofline_frac (bench.py N=1 C2)" > $out
for t in 0 256 0 256 0 256; do
  line=$(timeout 200 python bench.py --threads $t 2>/dev/null | tail -1)
  echo "$t $(python -c "import json,sys; d=json.loads(sys.argv[1]); print(d['value'], d['kernels_ms']['put_avg'], d['roofline']['frac'])" "$line")" >> $out
done
