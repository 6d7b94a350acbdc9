OUT=gpurun_out; mkdir -p $OUT
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 600 $TR --nproc-per-node 2 --master-port 29531 bench.py --gpus 2 --comm host --steps 30 --warmup 3 > $OUT/bench_n2_r2h.json 2> $OUT/bench_n2_r2h.err; echo "exit $?" >> $OUT/bench_n2_r2h.err
timeout 600 python bench.py --steps 100 --warmup 10 > $OUT/bench_n1_r2h.json 2> $OUT/bench_n1_r2h.err; echo "exit $?" >> $OUT/bench_n1_r2h.err
timeout 2400 python -m pytest tests -q -m gpu > $OUT/pytest_all_r2h.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_all_r2h.log
echo done
