# C4: TMA-fed CSR-stream variants vs the LSU CSR-stream kernel; C2/C3 regression check; remaining new GPU tests
OUT=gpurun_out; mkdir -p $OUT
f=$OUT/c4_variants_r2d.txt; : > $f
for cfg in "0 0" "1 0" "1 1" "1 2" "1 3"; do set -- $cfg
  r=$(DSPMV_STREAM_TMA=$1 DSPMV_STMA_VARIANT=$2 timeout 180 python bench.py --workload c4 --secondary none --steps 30 --warmup 5 --no-sweep --no-cpu-baseline --execution host 2>>$OUT/c4_variants_r2d.err | tail -1)
  echo "tma=$1 variant=$2 $(echo "$r" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print("yL_ms", r["avg_launch_ms"], "frac", r["frac"], "kernel", r["kernel"], "parity", d["parity_ok"])' 2>&1)" >> $f
done
for w in c2 c3; do
  r=$(timeout 300 python bench.py --workload $w --secondary none --steps 50 --warmup 5 --no-sweep --no-cpu-baseline 2>>$OUT/c4_variants_r2d.err | tail -1)
  echo "$w $(echo "$r" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print("yL_ms", r["avg_launch_ms"], "frac", r["frac"], "step_ms", d["ms_per_step"], "parity", d["parity_ok"])' 2>&1)" >> $f
done
timeout 1500 python -m pytest tests/test_gpu_boundary_opts.py tests/test_gpu_graph_exchange.py tests/test_gpu_oracle_sweeps.py -q -m gpu > $OUT/pytest_new_r2d.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_new_r2d.log
echo done
