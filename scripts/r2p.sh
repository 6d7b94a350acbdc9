OUT=gpurun_out; mkdir -p $OUT
f=$OUT/c4_ctawidth_r2p.txt; : > $f
for lib in "" w10 w20 "" w20; do
  r=$(DSPMV_LIB=$lib timeout 180 python bench.py --workload c4 --secondary none --steps 30 --warmup 5 --no-sweep --no-cpu-baseline --execution host 2>>$OUT/c4_ctawidth_r2p.err | tail -1)
  echo "lib=${lib:-w8} $(echo "$r" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print("yL_ms", r["avg_launch_ms"], "frac", r["frac"], "parity", d["parity_ok"])' 2>&1)" >> $f
done
echo done
