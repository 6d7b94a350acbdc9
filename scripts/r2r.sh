OUT=gpurun_out; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_boundary_opts.py tests/test_gpu_bench_contract.py -q -m gpu > $OUT/pytest_r2r.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_r2r.log
timeout 900 python bench.py --gpus 1 --steps 50 --warmup 5 > $OUT/bench_r2r.json 2> $OUT/bench_r2r.err; echo "bench exit $?" >> $OUT/bench_r2r.err
echo done
