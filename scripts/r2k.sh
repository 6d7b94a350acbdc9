OUT=gpurun_out; mkdir -p $OUT
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/ub_g4 scripts/ubench_tma_gather4.cu -lcuda > $OUT/ub_g4_r2k.txt 2>&1
for cfg in "2 1" "2 4" "4 1" "4 4" "8 1"; do set -- $cfg
  timeout 60 /tmp/ub_g4 134 64 $1 $2 1 >> $OUT/ub_g4_r2k.txt 2>&1; echo "exit $?" >> $OUT/ub_g4_r2k.txt
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_r2k.csv \
    python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-sweep > $OUT/ncu_launch_r2k.log 2>&1; echo "ncu1 exit $?" >> $OUT/ncu_launch_r2k.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"spmv_block" -s 3 -c 1 \
    -o $OUT/prof_c3_r2k -f python bench.py --workload c3 --secondary none --steps 2 --warmup 1 --no-cpu-baseline --no-sweep --execution host > $OUT/ncu_c3_r2k.log 2>&1; echo "exit $?" >> $OUT/ncu_c3_r2k.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"spmv_stream_kernel" -s 3 -c 1 \
    -o $OUT/prof_c4_r2k -f python bench.py --workload c4 --secondary none --steps 2 --warmup 1 --no-cpu-baseline --no-sweep --execution host > $OUT/ncu_c4_r2k.log 2>&1; echo "exit $?" >> $OUT/ncu_c4_r2k.log
echo done
