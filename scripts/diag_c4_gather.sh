#!/bin/bash
# C4's own gather pattern (its CSR col array, 134M ids) through ubench_gather_scope
OUT=gpurun_out; mkdir -p $OUT
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 scripts/ubench_gather_scope.cu -o /tmp/ugs || exit 1
python -c "
import gen
n, (rp, col, val) = gen.config_matrix('c4')
col.astype('int32').tofile('/tmp/c4col.bin')
print(n, len(col))
" > $OUT/c4col.log 2>&1
timeout 600 /tmp/ugs /tmp/c4col.bin > $OUT/ugs_c4pattern.txt 2>&1
