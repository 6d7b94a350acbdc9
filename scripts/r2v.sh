OUT=gpurun_out; mkdir -p $OUT
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_r2v.log 2>&1; echo "smoke exit $?" >> $OUT/smoke_r2v.log
timeout 2400 python -m pytest tests -q -m gpu > $OUT/pytest_all_r2v.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_all_r2v.log
timeout 900 python bench.py --gpus 1 > $OUT/bench_r2v.json 2> $OUT/bench_r2v.err; echo "bench exit $?" >> $OUT/bench_r2v.err
timeout 600 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $OUT/bench_ref_r2v.json 2> $OUT/bench_ref_r2v.err; echo "exit $?" >> $OUT/bench_ref_r2v.err
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 $TR --nproc-per-node 2 --master-port 29571 bench.py --gpus 2 --comm host --steps 30 --warmup 3 > $OUT/bench_n2_r2v.json 2> $OUT/bench_n2_r2v.err; echo "exit $?" >> $OUT/bench_n2_r2v.err
echo done
