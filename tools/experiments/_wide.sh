#!/bin/bash
OUT=gpurun_out/wide; mkdir -p $OUT
for i in 1 2; do
timeout 600 python bench.py --steps 30 --warmup 5 > $OUT/bench_16_$i.log 2>&1
ACCUDNN_REDUCE_WIDE=4 timeout 600 python bench.py --steps 30 --warmup 5 > $OUT/bench_4_$i.log 2>&1
ACCUDNN_REDUCE_WIDE=8 timeout 600 python bench.py --steps 30 --warmup 5 > $OUT/bench_8_$i.log 2>&1
done
