#!/bin/bash
# y_L block-config sweep on one workload: sweep_cfg_list.sh <workload> <cfg>...
OUT=gpurun_out; mkdir -p $OUT
w=$1; shift
for c in "$@"; do
  DSPMV_BLOCK_CFG=$c timeout 300 python bench.py --workload $w --steps 50 --warmup 5 --no-cpu-baseline --no-sweep \
      > $OUT/sw_${w}_cfg$c.json 2> $OUT/sw_${w}_cfg$c.err
  python -c "
import json,sys
d=json.loads(open('$OUT/sw_${w}_cfg$c.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$w cfg$c', 'yL_ms', r['avg_launch_ms'], 'GB/s', r['achieved'], 'frac', r['frac'], 'step_ms', d['ms_per_step'])" >> $OUT/sweep_${w}.txt 2>&1 || echo "$w cfg$c failed" >> $OUT/sweep_${w}.txt
done
