#!/bin/bash
# CSR-stream grid sweep on C4 (CTAs per SM, capped by occupancy)
OUT=gpurun_out; mkdir -p $OUT
for c in 5; do
  DSPMV_STREAM_CTAS=$c timeout 300 python bench.py --workload c4 --steps 50 --warmup 5 --no-cpu-baseline --no-sweep --execution host > $OUT/ss_$c.json 2>/dev/null
  python -c "
import json
d=json.loads(open('$OUT/ss_$c.json').read().strip().splitlines()[-1]); r=d['roofline']
print('c4 stream ctas/SM $c', 'yL_ms', r['avg_launch_ms'], 'GB/s', r['achieved'], 'frac', r['frac'], r['kernel'])" >> $OUT/sweep_stream.txt
done
