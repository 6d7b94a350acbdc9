OUT=gpurun_out; mkdir -p $OUT
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 420 $TR --nproc-per-node 2 --master-port 29521 bench.py --gpus 2 --comm host --steps 30 --warmup 3 > $OUT/bench_n2_r2g.json 2> $OUT/bench_n2_r2g.err; echo "exit $?" >> $OUT/bench_n2_r2g.err
timeout 600 python scripts/c5_exec_modes.py --out $OUT/r2_c5_exec_modes.json > $OUT/c5_exec_r2g.log 2>&1; echo "exit $?" >> $OUT/c5_exec_r2g.log
f=$OUT/e2e_chunks_r2g.txt; : > $f
for k in 4 8 16 32; do
  r=$(DSPMV_HOST_CHUNKS=$k timeout 300 python bench.py --workload c3 --secondary none --steps 20 --warmup 3 --no-sweep --no-cpu-baseline 2>>$OUT/e2e_chunks_r2g.err | tail -1)
  echo "chunks=$k $(echo "$r" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); e=d["e2e"]; print("e2e_ms", e["ms_per_step"], "pcie_frac", e["pcie"]["pcie_frac"], "floor_ms", e["pcie"]["copy_floor_ms"])' 2>&1)" >> $f
done
timeout 1200 python -m pytest tests/test_gpu_bench_contract.py -q -m gpu > $OUT/pytest_bench_r2g.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_bench_r2g.log
echo done
