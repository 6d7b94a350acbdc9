#!/bin/bash
OUT=gpurun_out; TAG=${1:-c4}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"spmv_(block|vector)" -s 4 -c 2 \
    -o $OUT/prof_$TAG -f python bench.py --workload c4 --steps 3 --warmup 2 --no-cpu-baseline --no-sweep > $OUT/ncu_$TAG.log 2>&1
echo "ncu exit $?" >> $OUT/ncu_$TAG.log
