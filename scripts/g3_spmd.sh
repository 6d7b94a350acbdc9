OUT=gpurun_out; mkdir -p $OUT
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 1500 $TR --nproc-per-node 4 --master-port 29581 scripts/design_rules.py --workload g3 --comm host --syncs derived \
   --resume $OUT/rules_g3_der.jsonl --out $OUT/r2_rules_g3_4proc_derived.json > $OUT/rules_g3_der.log 2>&1; echo "exit $?" >> $OUT/rules_g3_der.log
timeout 2400 $TR --nproc-per-node 4 --master-port 29582 scripts/design_rules.py --workload g3 --comm host --syncs orderable \
   --resume $OUT/rules_g3_ord.jsonl --out $OUT/r2_rules_g3_4proc_orderable.json > $OUT/rules_g3_ord.log 2>&1; echo "exit $?" >> $OUT/rules_g3_ord.log
echo done
