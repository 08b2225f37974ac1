#!/bin/bash
# Same-box A/B of the N=2 ring-of-pairs line vs put threads per CTA (33 CTAs).
out=gpurun_out/pairs_ab.txt
echo "# threads value_GBps_total roofline_frac (bench.py --gpus 2, pairs)" > $out
p=29600
for t in 0 480 448 0 480 448; do
  p=$((p+1))
  line=$(timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $p bench.py --gpus 2 --threads $t --lat-iters 60 2>/dev/null | grep '^{' | tail -1)
  echo "$t $(python -c "import json,sys; d=json.loads(sys.argv[1]); print(d['value'], d['roofline']['frac'])" "$line" 2>/dev/null)" >> $out
done
