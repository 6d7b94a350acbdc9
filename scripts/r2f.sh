# multi-process (SPMD) runs on one B200: C5 orderable sweep over 4 processes, design rules from SPMD
# processes, the N=2 bench path; then the whole GPU suite
OUT=gpurun_out; mkdir -p $OUT
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 $TR --nproc-per-node 4 --master-port 29511 bench.py --gpus 4 --workload c5 --comm host --space orderable \
   --sweep-out $OUT/r2_sweep_c5_4proc.json --secondary none --steps 50 --warmup 5 > $OUT/bench_c5_4proc_r2f.json 2> $OUT/bench_c5_4proc_r2f.err; echo "exit $?" >> $OUT/bench_c5_4proc_r2f.err
timeout 600 $TR --nproc-per-node 2 --master-port 29512 bench.py --gpus 2 --comm host --steps 30 --warmup 3 > $OUT/bench_n2_r2f.json 2> $OUT/bench_n2_r2f.err; echo "exit $?" >> $OUT/bench_n2_r2f.err
timeout 1200 $TR --nproc-per-node 4 --master-port 29513 scripts/design_rules.py --workload c5 --comm host --syncs orderable \
   --out $OUT/r2_rules_c5_4proc_ord.json > $OUT/rules_c5_r2f.log 2>&1; echo "exit $?" >> $OUT/rules_c5_r2f.log
timeout 1800 python -m pytest tests -q -m gpu -x > $OUT/pytest_all_r2f.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_all_r2f.log
echo done
