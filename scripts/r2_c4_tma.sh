# C4 y_L: CSR-stream (LSU) vs CSR-stream with a TMA producer, with/without an L2 persisting window on x
OUT=gpurun_out; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "stream" > $OUT/pytest_stream_r2b.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_stream_r2b.log
f=$OUT/c4_tma_r2b.txt; : > $f
for cfg in "0 0" "1 0" "1 0.5" "1 1.0" "0 1.0"; do set -- $cfg
  r=$(DSPMV_STREAM_TMA=$1 DSPMV_X_PERSIST=$2 timeout 300 python bench.py --workload c4 --steps 20 --warmup 5 --no-sweep --no-cpu-baseline 2>>$OUT/c4_tma_r2b.err | tail -1)
  echo "tma=$1 persist=$2 $(echo "$r" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print("yL_ms", r["avg_launch_ms"], "frac", r["frac"], "kernel", r["kernel"])')" >> $f
done
DSPMV_STREAM_TMA=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"spmv_stream" -s 2 -c 1 \
    -o $OUT/prof_c4_tma_r2b -f python bench.py --workload c4 --steps 2 --warmup 1 --no-cpu-baseline --no-sweep > $OUT/ncu_c4_tma_r2b.log 2>&1
echo done
