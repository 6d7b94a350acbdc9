#!/bin/bash
# Sweep the row-block kernel configurations (y_L only, no schedule sweep).
W=${1:-c2}; TAG=${2:-sw}
OUT=gpurun_out; mkdir -p $OUT
for c in 0 1 2 3 4 5 6 7; do
  DSPMV_BLOCK_CFG=$c timeout 300 python bench.py --workload $W --steps 200 --warmup 20 --no-cpu-baseline --no-sweep > $OUT/${TAG}_${W}_cfg$c.json 2> /dev/null
done
python - "$W" "$TAG" <<'PY'
import json, sys
w, tag = sys.argv[1], sys.argv[2]
for c in range(8):
    try:
        d = json.loads(open(f'gpurun_out/{tag}_{w}_cfg{c}.json').read().strip().splitlines()[-1])
        r = d['roofline']; print(w, 'cfg', c, r['avg_launch_ms'], r['achieved'], r['frac'])
    except Exception as e:
        print(w, 'cfg', c, 'ERR', e)
PY
