OUT=gpurun_out; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $OUT/gpu_r2a.txt 2>&1
nproc >> $OUT/gpu_r2a.txt
timeout 1500 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu_r2a.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu_r2a.log
for w in c3 c4; do
( time timeout 600 python bench.py --workload $w --steps 20 --warmup 5 --no-sweep --no-cpu-baseline ) > $OUT/bench_${w}_r2a.json 2> $OUT/bench_${w}_r2a.err
done
echo done
