#!/bin/bash
# BN L2 keep thresholds re-measured on the final kernels
OUT=gpurun_out/keep2; mkdir -p $OUT
for i in 1 2; do
  timeout 600 python bench.py --steps 30 --warmup 5 > $OUT/bench_def_$i.log 2>&1
  ACCUDNN_BN_KEEP_MB_BWD=96 timeout 600 python bench.py --steps 30 --warmup 5 > $OUT/bench_b96_$i.log 2>&1
  ACCUDNN_BN_KEEP_MB_FWD=64 timeout 600 python bench.py --steps 30 --warmup 5 > $OUT/bench_f64_$i.log 2>&1
  ACCUDNN_BN_KEEP_MB_BWD=56 timeout 600 python bench.py --steps 30 --warmup 5 > $OUT/bench_b56_$i.log 2>&1
done
