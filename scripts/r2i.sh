OUT=gpurun_out; mkdir -p $OUT
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 200 $TR --nproc-per-node 2 --master-port 29541 scripts/repro_put_e2e.py c2 > $OUT/repro_c2_r2i.log 2>&1; echo "exit $?" >> $OUT/repro_c2_r2i.log
timeout 200 $TR --nproc-per-node 2 --master-port 29542 scripts/repro_put_e2e.py c3 > $OUT/repro_c3_r2i.log 2>&1; echo "exit $?" >> $OUT/repro_c3_r2i.log
DSPMV_HOST_CHUNKS=4 timeout 200 $TR --nproc-per-node 2 --master-port 29543 scripts/repro_put_e2e.py c3 > $OUT/repro_c3k4_r2i.log 2>&1; echo "exit $?" >> $OUT/repro_c3k4_r2i.log
timeout 200 $TR --nproc-per-node 2 --master-port 29544 scripts/repro_put_e2e.py c3 graph > $OUT/repro_c3g_r2i.log 2>&1; echo "exit $?" >> $OUT/repro_c3g_r2i.log
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/ub_g4 scripts/ubench_tma_gather4.cu -lcuda > $OUT/ub_g4_r2i.txt 2>&1
timeout 120 /tmp/ub_g4 134 64 >> $OUT/ub_g4_r2i.txt 2>&1; echo "exit $?" >> $OUT/ub_g4_r2i.txt
timeout 120 /tmp/ub_g4 134 8 >> $OUT/ub_g4_r2i.txt 2>&1; echo "exit $?" >> $OUT/ub_g4_r2i.txt
echo done
