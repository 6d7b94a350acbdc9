OUT=gpurun_out; mkdir -p $OUT
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/uz scripts/ubench_zerocopy.cu > $OUT/uz_r2s.txt 2>&1
timeout 120 /tmp/uz 134 >> $OUT/uz_r2s.txt 2>&1; echo "exit $?" >> $OUT/uz_r2s.txt
timeout 1200 python -m pytest tests/test_gpu_graph_exchange.py -q -m gpu -k full_size > $OUT/pytest_full_r2s.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_full_r2s.log
echo done
