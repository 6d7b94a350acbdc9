#!/bin/bash
# One GPU round trip: smoke, GPU tests, bench (ours + reference), ncu launch
# list + full captures of the y_L kernel on C2/C3/C4.
TAG=${1:-r1}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $OUT/gpu_$TAG.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke exit $?" >> $OUT/smoke_$TAG.log
timeout 1800 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu_$TAG.log
timeout 900 python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; echo "bench exit $?" >> $OUT/bench_$TAG.err
timeout 300 python bench.py --impl reference --steps 20 --warmup 2 > $OUT/bench_ref_$TAG.json 2> $OUT/bench_ref_$TAG.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$TAG.csv \
    python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-sweep > $OUT/ncu_launch_$TAG.log 2>&1; echo "ncu1 exit $?" >> $OUT/ncu_launch_$TAG.log
for w in c2 c3 c4; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"spmv_(block|stream)" -s 2 -c 1 \
    -o $OUT/prof_${w}_$TAG -f python bench.py --workload $w --steps 2 --warmup 1 --no-cpu-baseline --no-sweep > $OUT/ncu_full_${w}_$TAG.log 2>&1; echo "ncu $w exit $?" >> $OUT/ncu_full_${w}_$TAG.log
done
echo done
