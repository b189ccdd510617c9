#!/bin/bash
OUT=gpurun_out/keep; mkdir -p $OUT
for i in 1 2; do
timeout 600 python bench.py --steps 30 --warmup 5 > $OUT/bench_def_$i.log 2>&1
ACCUDNN_BN_KEEP_MB_BWD=48 timeout 600 python bench.py --steps 30 --warmup 5 > $OUT/bench_b48_$i.log 2>&1
ACCUDNN_BN_KEEP_MB_BWD=100 timeout 600 python bench.py --steps 30 --warmup 5 > $OUT/bench_b100_$i.log 2>&1
ACCUDNN_BN_KEEP_MB_FWD=72 timeout 600 python bench.py --steps 30 --warmup 5 > $OUT/bench_f72_$i.log 2>&1
done
for i in 1 2; do ACCUDNN_REDUCE_WIDE=1000 timeout 600 python bench.py --steps 30 --warmup 5 > $OUT/bench_nowide_$i.log 2>&1; done
