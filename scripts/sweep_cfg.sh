#!/bin/bash
# Sweep the row-block kernel configurations on the C2 bench (1 GPU).
TAG=${1:-sweep}
OUT=gpurun_out; mkdir -p $OUT
for c in 0 1 2 3 4 5; do
  DSPMV_BLOCK_CFG=$c timeout 300 python bench.py --steps 300 --warmup 20 --no-cpu-baseline > $OUT/${TAG}_cfg$c.json 2> $OUT/${TAG}_cfg$c.err
done
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/*_cfg*.json')):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        r=d['roofline']; print(f, d['value'], d['ms_per_step'], r['avg_launch_ms'], r['achieved'], r['frac'])
    except Exception as e: print(f, 'ERR', e)
PY
