#!/bin/bash
# L2 hit rate of C4's gather pattern alone (ubench_gather_scope file mode, evict_last hint,
# 32 warps/SM, L2 flushed) for comparison with the y_L kernel's x lookups
OUT=gpurun_out; mkdir -p $OUT
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 scripts/ubench_gather_scope.cu -o /tmp/ugs || exit 1
python -c "
import gen
n, (rp, col, val) = gen.config_matrix('c4')
col.astype('int32').tofile('/tmp/c4col.bin')
"
M=lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum,lts__t_sectors_srcunit_tex_op_read_evict_last_lookup_hit.sum,lts__t_sectors_srcunit_tex_op_read_evict_last_lookup_miss.sum,dram__bytes_read.sum,gpu__time_duration.sum
timeout 600 ncu --metrics $M --cache-control none --clock-control none -k regex:ldg_kernel --launch-skip 51 --launch-count 3 --csv /tmp/ugs /tmp/c4col.bin > $OUT/ncu_ubench_c4.csv 2>&1
