#!/bin/bash
# apply_host x chunking on C2: uniform 4 chunks vs front-loaded splits (DSPMV_HOST_SPLIT)
OUT=gpurun_out; mkdir -p $OUT
for sp in "" "0.3,0.55,0.75,0.9,0.97" "0.25,0.5,0.7,0.85,0.95,0.99" "0.2,0.4,0.6,0.75,0.87,0.95,0.99"; do
  DSPMV_HOST_SPLIT=$sp timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline > $OUT/hs.json 2>/dev/null
  python -c "
import json
d=json.loads(open('$OUT/hs.json').read().strip().splitlines()[-1]); e=d['e2e']
print('split=[$sp]', 'e2e_ms', e['ms_per_step'], 'GFLOP/s', e['value'])" >> $OUT/host_split.txt
done
