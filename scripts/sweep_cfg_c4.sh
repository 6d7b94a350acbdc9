#!/bin/bash
OUT=gpurun_out; mkdir -p $OUT
for c in 0 1 2 3 4 5; do
  DSPMV_BLOCK_CFG=$c timeout 300 python bench.py --workload ${1:-c4} --steps 50 --warmup 5 --no-cpu-baseline --no-sweep > $OUT/sw${1:-c4}_cfg$c.json 2> $OUT/sw${1:-c4}_cfg$c.err
done
