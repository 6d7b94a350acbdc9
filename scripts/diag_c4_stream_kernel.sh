#!/bin/bash
# C4 through a CSR-stream kernel: scripts/ubench_csr_stream.cu
OUT=gpurun_out; mkdir -p $OUT
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 scripts/ubench_csr_stream.cu -o /tmp/ucst || exit 1
python -c "
import gen, numpy as np
n, (rp, col, val) = gen.config_matrix('c4')
rp.astype('int32').tofile('/tmp/c4rp.bin'); col.astype('int32').tofile('/tmp/c4col.bin'); val.astype('float64').tofile('/tmp/c4val.bin')
"
timeout 300 /tmp/ucst > $OUT/ucst.txt 2>&1
