#!/bin/bash
# y_L time per workload (auto block config unless CFG_<w> is set): quick_yl.sh <tag> <workload>...
OUT=gpurun_out; mkdir -p $OUT
tag=$1; shift
for w in "$@"; do
  timeout 300 python bench.py --workload $w --steps 50 --warmup 5 --no-cpu-baseline --no-sweep --execution host \
      > $OUT/q_${tag}_$w.json 2> $OUT/q_${tag}_$w.err
  python -c "
import json
d=json.loads(open('$OUT/q_${tag}_$w.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$tag $w', 'yL_ms', r['avg_launch_ms'], 'GB/s', r['achieved'], 'frac', r['frac'])" >> $OUT/quick_yl.txt 2>&1 || echo "$tag $w failed" >> $OUT/quick_yl.txt
done
