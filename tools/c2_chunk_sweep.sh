#!/bin/bash
# C2 bench vs unit size (B200RING_CHUNK) and threads per CTA, same box.
out=gpurun_out/c2_chunk_sweep.txt
echo "# chunk threads value_GBps put_avg_ms roofline_frac (bench.py N=1 C2)" > $out
for cfg in "32768 224" "16384 224" "65536 224" "16384 192" "65536 448" "32768 224" "16384 224"; do
  set -- $cfg
  line=$(B200RING_CHUNK=$1 timeout 200 python bench.py --threads $2 2>/dev/null | tail -1)
  echo "$1 $2 $(python -c "import json,sys; d=json.loads(sys.argv[1]); print(d['value'], d['kernels_ms']['put_avg'], d['roofline']['frac'])" "$line" 2>/dev/null)" >> $out
done
