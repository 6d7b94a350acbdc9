#!/bin/bash
# CSR-stream kernel forced (DSPMV_SKERNEL=2) on the stencil configs vs their auto row-block kernel
OUT=gpurun_out; mkdir -p $OUT
for w in c2 c3; do for k in 0 2; do
  DSPMV_SKERNEL=$k timeout 600 python bench.py --workload $w --steps 30 --warmup 5 --no-cpu-baseline --no-sweep --execution host > $OUT/sk_${w}_$k.json 2>/dev/null
  python -c "
import json
d=json.loads(open('$OUT/sk_${w}_$k.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$w skernel_env=$k', 'yL_ms', r['avg_launch_ms'], 'frac', r['frac'], r['kernel'])" >> $OUT/stream_stencils.txt
done; done
