#!/bin/bash
# C4 y_L with the gather removed (diag1) or made row-local (diag2) vs the product build
OUT=gpurun_out; mkdir -p $OUT
for v in "" diag1 diag2; do
  DSPMV_LIB=$v DSPMV_BLOCK_CFG=3 timeout 300 python bench.py --workload c4 --steps 50 --warmup 5 --no-cpu-baseline --no-sweep --execution host > $OUT/gc_$v.json 2> $OUT/gc_$v.err
  python -c "
import json
d=json.loads(open('$OUT/gc_$v.json').read().strip().splitlines()[-1]); r=d['roofline']
print('c4 lib=$v', 'yL_ms', r['avg_launch_ms'], 'GB/s', r['achieved'])" >> $OUT/gather_cost.txt 2>&1
done
