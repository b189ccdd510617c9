#!/bin/bash
OUT=gpurun_out/ab1; mkdir -p $OUT
B="python bench.py --steps 30 --warmup 5"
for i in 1 2; do
timeout 600 $B > $OUT/head_$i.log 2>&1
cp profiles/b200/conv_tune.txt /tmp/tune_head.txt
cp _ab/tune_7d05672.txt profiles/b200/conv_tune.txt; timeout 600 $B > $OUT/head_tune7d_$i.log 2>&1
cp _ab/tune_r1.txt profiles/b200/conv_tune.txt; timeout 600 $B > $OUT/head_tuner1_$i.log 2>&1
cp /tmp/tune_head.txt profiles/b200/conv_tune.txt
(cd _ab/r1 && timeout 600 $B > ../../$OUT/r1_$i.log 2>&1)
done
timeout 300 python tools/swap_trace.py resnet20 32 12 8 8 plan $OUT/r20 > $OUT/r20.log 2>&1
grep -h -o '"value": [0-9.]*' $OUT/*.log
