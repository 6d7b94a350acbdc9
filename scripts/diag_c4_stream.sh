#!/bin/bash
OUT=gpurun_out; mkdir -p $OUT
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 scripts/ubench_gather_stream.cu -o /tmp/ugst || exit 1
python -c "
import gen
n, (rp, col, val) = gen.config_matrix('c4')
col.astype('int32').tofile('/tmp/c4col.bin')
"
timeout 300 /tmp/ugst /tmp/c4col.bin g > $OUT/ugst2.txt 2>&1
