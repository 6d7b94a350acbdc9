# round-2 check: new GPU tests, C4 kernel/persist experiment, default bench, ncu of the TMA-fed kernel
OUT=gpurun_out; mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_boundary_opts.py tests/test_gpu_graph_exchange.py tests/test_gpu_oracle_sweeps.py -x -q -m gpu > $OUT/pytest_new_r2c.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_new_r2c.log
f=$OUT/c4_persist_r2c.txt; : > $f
for cfg in "0 0" "0 1.0" "1 0" "1 1.0"; do set -- $cfg
  r=$(DSPMV_STREAM_TMA=$1 DSPMV_X_PERSIST=$2 timeout 180 python bench.py --workload c4 --secondary none --steps 20 --warmup 5 --no-sweep --no-cpu-baseline --execution host 2>>$OUT/c4_persist_r2c.err | tail -1)
  echo "tma=$1 persist=$2 $(echo "$r" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print("yL_ms", r["avg_launch_ms"], "frac", r["frac"], "kernel", r["kernel"], "parity", d["parity_ok"])' 2>&1)" >> $f
done
timeout 900 python bench.py --steps 50 --warmup 5 > $OUT/bench_default_r2c.json 2> $OUT/bench_default_r2c.err; echo "bench exit $?" >> $OUT/bench_default_r2c.err
DSPMV_STREAM_TMA=1 timeout 400 ncu --set full --clock-control none --import-source on -k regex:"spmv_stream_tma" -s 2 -c 1 \
    -o $OUT/prof_c4_tma_r2c -f python bench.py --workload c4 --secondary none --steps 2 --warmup 1 --no-cpu-baseline --no-sweep --execution host > $OUT/ncu_c4_tma_r2c.log 2>&1
echo done
