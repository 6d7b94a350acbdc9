# C4 y_L: CSR-stream kernel with the row indices prefetched (5 CTAs/SM capped regs, 4 CTAs/SM),
# TMA-fed variants with prefetched out[]; C2/C3 after the coherent-load instantiation split; PCIe peak
OUT=gpurun_out; mkdir -p $OUT
f=$OUT/c4_variants_r2e.txt; : > $f
one() {  # label env...
  lab=$1; shift
  r=$(env "$@" timeout 180 python bench.py --workload c4 --secondary none --steps 30 --warmup 5 --no-sweep --no-cpu-baseline --execution host 2>>$OUT/c4_variants_r2e.err | tail -1)
  echo "$lab $(echo "$r" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print("yL_ms", r["avg_launch_ms"], "frac", r["frac"], "kernel", r["kernel"], "parity", d["parity_ok"])' 2>&1)" >> $f
}
one k1b_mc5 DSPMV_STREAM_TMA=0
one k1b_mc4 DSPMV_STREAM_TMA=0 DSPMV_LIB=mc4
one tma_v0 DSPMV_STREAM_TMA=1 DSPMV_STMA_VARIANT=0
one tma_v1 DSPMV_STREAM_TMA=1 DSPMV_STMA_VARIANT=1
one tma_v2 DSPMV_STREAM_TMA=1 DSPMV_STMA_VARIANT=2
for w in c2 c3; do
  r=$(timeout 300 python bench.py --workload $w --secondary none --steps 50 --warmup 5 --no-sweep --no-cpu-baseline 2>>$OUT/c4_variants_r2e.err | tail -1)
  echo "$w $(echo "$r" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print("yL_ms", r["avg_launch_ms"], "frac", r["frac"], "step_ms", d["ms_per_step"], "parity", d["parity_ok"])' 2>&1)" >> $f
done
timeout 120 python scripts/pcie_peak.py > $OUT/pcie_r2e.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_apply_host.py -q -m gpu -k "stream or apply_host" > $OUT/pytest_stream_r2e.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_stream_r2e.log
echo done
