#!/bin/bash
# CSR-stream with TMA-staged col/val (DSPMV_STREAM_TMA=1) vs the product kernel on C4, + parity.
# The TMA variant was measured (profiles/r1_stream_kernel_c4_sweep.txt) and removed; the knob is now a no-op.
OUT=gpurun_out; mkdir -p $OUT
DSPMV_STREAM_TMA=1 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "stream or irregular" > $OUT/pytest_tma.log 2>&1; echo "exit $?" >> $OUT/pytest_tma.log
for v in 0 1; do
  DSPMV_STREAM_TMA=$v timeout 300 python bench.py --workload c4 --steps 50 --warmup 5 --no-cpu-baseline --no-sweep --execution host > $OUT/tma_$v.json 2>/dev/null
  python -c "
import json
d=json.loads(open('$OUT/tma_$v.json').read().strip().splitlines()[-1]); r=d['roofline']
print('c4 stream_tma=$v', 'yL_ms', r['avg_launch_ms'], 'GB/s', r['achieved'])" >> $OUT/stream_tma.txt
done
