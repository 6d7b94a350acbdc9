# integrated check: smoke, whole GPU suite, default bench (driver command), reference arm
OUT=gpurun_out; mkdir -p $OUT
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_r2q.log 2>&1; echo "smoke exit $?" >> $OUT/smoke_r2q.log
timeout 2400 python -m pytest tests -q -m gpu > $OUT/pytest_all_r2q.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_all_r2q.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > $OUT/bench_r2q.json 2> $OUT/bench_r2q.err; echo "bench exit $?" >> $OUT/bench_r2q.err
timeout 600 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $OUT/bench_ref_r2q.json 2> $OUT/bench_ref_r2q.err; echo "exit $?" >> $OUT/bench_ref_r2q.err
echo done
