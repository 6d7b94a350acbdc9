OUT=gpurun_out; mkdir -p $OUT
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/ub_g4 scripts/ubench_tma_gather4.cu -lcuda > $OUT/ub_g4_r2m.txt 2>&1
echo "# mode 3: plain 2-D tile load control (1 of the 4 indices per lane fetched; the rate line counts all 4)" >> $OUT/ub_g4_r2m.txt
timeout 60 /tmp/ub_g4 134 64 2 1 3 >> $OUT/ub_g4_r2m.txt 2>&1; echo "exit $?" >> $OUT/ub_g4_r2m.txt
timeout 60 /tmp/ub_g4 134 64 4 1 3 >> $OUT/ub_g4_r2m.txt 2>&1; echo "exit $?" >> $OUT/ub_g4_r2m.txt
echo done
