#!/bin/bash
# Reproduces round 2's GPU evidence on one B200 (gpurun --timeout 5400 -- 'bash scripts/gpu_round2.sh [what]'):
#   check    smoke, the whole -m gpu suite, the driver's bench command, the reference arm
#   multi    bench.py's N>1 path as 2 processes on one GPU, the C5 sweep as 4 SPMD processes,
#            design rules from the SPMD dataset, the C5 execution-model comparison
#   profile  ncu launch list of the default bench, full captures of the C3 / C4 y_L kernels,
#            compute-sanitizer over scripts/sanitize.py
#   ubench   PCIe peak, zero-copy stores, LSU vs TMA random gathers
#   kernels  the round-2 y_L sweeps: L2 prefetch distance (C3, C2), K1b hand-out and K1d settings (C4),
#            column panels (C4) -- profiles/r2_l2_prefetch.txt, r2_c4_sell.txt
# Outputs land in gpurun_out/ (summaries are copied to profiles/ by hand).
set -u
OUT=gpurun_out; mkdir -p $OUT
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
what=${1:-check}
case $what in
check)
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke exit $?" >> $OUT/smoke.log
  timeout 2400 python -m pytest tests -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu.log
  timeout 900 python bench.py --gpus 1 > $OUT/bench.json 2> $OUT/bench.err; echo "bench exit $?" >> $OUT/bench.err
  timeout 600 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
  ;;
multi)
  timeout 900 $TR --nproc-per-node 2 --master-port 29571 bench.py --gpus 2 --comm host --steps 30 --warmup 3 \
      > $OUT/bench_n2.json 2> $OUT/bench_n2.err
  timeout 900 $TR --nproc-per-node 4 --master-port 29572 bench.py --gpus 4 --workload c5 --comm host --space orderable \
      --sweep-out $OUT/sweep_c5_4proc.json --secondary none --steps 50 --warmup 5 > $OUT/bench_c5_4proc.json 2> $OUT/bench_c5_4proc.err
  timeout 1200 $TR --nproc-per-node 4 --master-port 29573 scripts/design_rules.py --workload c5 --comm host --syncs orderable \
      --resume $OUT/rules_c5_sweep.jsonl --out $OUT/rules_c5_4proc_orderable.json > $OUT/rules_c5.log 2>&1
  timeout 600 python scripts/c5_exec_modes.py --out $OUT/c5_exec_modes.json > $OUT/c5_exec_modes.log 2>&1
  ;;
profile)
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
      python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-sweep > $OUT/ncu_launch.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"spmv_block" -s 3 -c 1 -o $OUT/prof_c3 -f \
      python bench.py --workload c3 --secondary none --steps 2 --warmup 1 --no-cpu-baseline --no-sweep --execution host > $OUT/ncu_c3.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"spmv_stream_kernel" -s 3 -c 1 -o $OUT/prof_c4 -f \
      python bench.py --workload c4 --secondary none --steps 2 --warmup 1 --no-cpu-baseline --no-sweep --execution host > $OUT/ncu_c4.log 2>&1
  for tool in memcheck racecheck synccheck; do  # the pool may close compute-sanitizer (exit 86)
    timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 python scripts/sanitize.py > $OUT/san_$tool.log 2>&1
    echo "$tool exit $?" >> $OUT/sanitizer.txt
  done
  ;;
ubench)
  timeout 120 python scripts/pcie_peak.py > $OUT/pcie.txt 2>&1
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/uz scripts/ubench_zerocopy.cu && timeout 120 /tmp/uz 134 > $OUT/uz.txt 2>&1
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/ug scripts/ubench_tma_gather4.cu -lcuda && \
      { timeout 60 /tmp/ug 134 64 2 1 0; timeout 60 /tmp/ug 134 64 2 1 3; timeout 60 /tmp/ug 134 64 2 1 1; } > $OUT/ug.txt 2>&1
  ;;
kernels)
  S="timeout 600 python scripts/sell_sweep.py --reps 30"
  for w in c3 c2; do $S --workload $w --cfgs auto:0,auto:1,auto:2,auto:4 > $OUT/l2pf_$w.txt 2>&1; done
  for d in 0 1; do DSPMV_ST_DYNAMIC=$d $S --workload c4 --cfgs stream,stream > $OUT/c4_dyn$d.txt 2>&1; done
  $S --workload c4 --cfgs stream,sell:256:4:64:2048:6,sell:256:4:256:2048:6,sell:256:4:64:4096:6 > $OUT/c4_sell.txt 2>&1
  $S --workload c4 --long-row-sum 1 --cfgs stream,sell:256:4:64:2048:6 > $OUT/c4_stored.txt 2>&1
  timeout 900 python scripts/c4_panels.py > $OUT/c4_panels.txt 2>&1
  ;;
esac
echo done
