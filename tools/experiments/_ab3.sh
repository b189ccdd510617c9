#!/bin/bash
OUT=gpurun_out/ab3; mkdir -p $OUT
B="python bench.py --steps 30 --warmup 5"
cp profiles/b200/conv_tune.txt /tmp/tune_head.txt
for i in 1 2; do
cp /tmp/tune_head.txt profiles/b200/conv_tune.txt; timeout 600 $B > $OUT/head_$i.log 2>&1
cp _ab/tune_7d05672.txt profiles/b200/conv_tune.txt; timeout 600 $B > $OUT/t7d_$i.log 2>&1
cp _ab/tune_r1.txt profiles/b200/conv_tune.txt; timeout 600 $B > $OUT/tr1_$i.log 2>&1
done
cp /tmp/tune_head.txt profiles/b200/conv_tune.txt
