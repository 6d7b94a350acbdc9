#!/bin/bash
# C4 through a plain (unstaged) CSR kernel: scripts/ubench_csr_naive.cu
OUT=gpurun_out; mkdir -p $OUT
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 scripts/ubench_csr_naive.cu -o /tmp/ucsr || exit 1
python -c "
import gen, numpy as np
n, (rp, col, val) = gen.config_matrix('c4')
rp.astype('int32').tofile('/tmp/c4rp.bin'); col.astype('int32').tofile('/tmp/c4col.bin'); val.astype('float64').tofile('/tmp/c4val.bin')
"
timeout 300 /tmp/ucsr > $OUT/ucsr.txt 2>&1
