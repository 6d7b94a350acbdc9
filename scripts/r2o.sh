# C4 y_L diagnostics of the CSR-stream kernel (K1b): product, DIAG=3 (no row sums), DIAG=4 (no gathers),
# DIAG=5 (no shared memory), EF (matrix stream with an explicit L2 evict_first policy)
OUT=gpurun_out; mkdir -p $OUT
f=$OUT/c4_diag_r2o.txt; : > $f
for lib in "" diag3 diag4 diag5 ef "" ef; do
  r=$(DSPMV_LIB=$lib timeout 180 python bench.py --workload c4 --secondary none --steps 30 --warmup 5 --no-sweep --no-cpu-baseline --execution host 2>>$OUT/c4_diag_r2o.err | tail -1)
  echo "lib=${lib:-product} $(echo "$r" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print("yL_ms", r["avg_launch_ms"], "frac", r["frac"], "parity", d["parity_ok"])' 2>&1)" >> $f
done
echo done
