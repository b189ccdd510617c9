#!/bin/bash
OUT=gpurun_out/padd3; mkdir -p $OUT
cp profiles/b200/conv_tune.txt /tmp/t0.txt
for i in 1 2; do
cp /tmp/t0.txt profiles/b200/conv_tune.txt; timeout 600 python bench.py --steps 30 --warmup 5 > $OUT/bench_t0_$i.log 2>&1
cp _ab/tune_padd.txt profiles/b200/conv_tune.txt; timeout 600 python bench.py --steps 30 --warmup 5 > $OUT/bench_padd_$i.log 2>&1
done
cp /tmp/t0.txt profiles/b200/conv_tune.txt
