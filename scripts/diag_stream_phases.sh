#!/bin/bash
# CSR-stream kernel on C4: product vs no row sums (DIAG=3) vs no gathers (DIAG=1)
OUT=gpurun_out; mkdir -p $OUT
for v in ""; do
  DSPMV_LIB=$v timeout 300 python bench.py --workload c4 --steps 50 --warmup 5 --no-cpu-baseline --no-sweep --execution host > $OUT/sp_$v.json 2>/dev/null
  python -c "
import json
d=json.loads(open('$OUT/sp_$v.json').read().strip().splitlines()[-1]); r=d['roofline']
print('c4 lib=$v', 'yL_ms', r['avg_launch_ms'], 'GB/s', r['achieved'])" >> $OUT/stream_phases.txt
done
