OUT=gpurun_out; mkdir -p $OUT
timeout 300 python -m pytest tests/test_gpu_apply_host.py -q -m gpu -x > $OUT/pytest_ycopy_r2u.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_ycopy_r2u.log
f=$OUT/e2e_ycopy_r2u.txt; : > $f
for w in c3 c2; do for yc in 1 0 1 0; do
  r=$(DSPMV_HOST_YCOPY=$yc timeout 240 python bench.py --workload $w --secondary none --steps 30 --warmup 3 --no-sweep --no-cpu-baseline 2>>$OUT/e2e_ycopy_r2u.err | tail -1)
  echo "$w ycopy=$yc $(echo "$r" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); e=d["e2e"]; print("e2e_ms", e["ms_per_step"], "GFLOP/s", e["value"], "pcie_frac", e["pcie"]["pcie_frac"], "parity", d["parity_ok"])' 2>&1 | tail -1)" >> $f
done; done
timeout 600 python -m pytest tests/test_gpu_multiproc_put.py tests/test_gpu_oracle_sweeps.py -q -m gpu -k "apply_host or multiprocess" > $OUT/pytest_ycopy2_r2u.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_ycopy2_r2u.log
echo done
