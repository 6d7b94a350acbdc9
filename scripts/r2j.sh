OUT=gpurun_out; mkdir -p $OUT
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for i in 1 2 3; do
timeout 200 $TR --nproc-per-node 2 --master-port 2955$i scripts/repro_put_e2e.py c3 graph > $OUT/repro_c3g${i}_r2j.log 2>&1; echo "exit $?" >> $OUT/repro_c3g${i}_r2j.log
done
timeout 600 $TR --nproc-per-node 2 --master-port 29559 bench.py --gpus 2 --comm host --steps 30 --warmup 3 > $OUT/bench_n2_r2j.json 2> $OUT/bench_n2_r2j.err; echo "exit $?" >> $OUT/bench_n2_r2j.err
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/ub_g4 scripts/ubench_tma_gather4.cu -lcuda > $OUT/ub_g4_r2j.txt 2>&1
timeout 120 /tmp/ub_g4 134 64 >> $OUT/ub_g4_r2j.txt 2>&1; echo "exit $?" >> $OUT/ub_g4_r2j.txt
echo done
