#!/bin/bash
OUT=gpurun_out/r2b; mkdir -p $OUT
timeout 900 python tools/table1.py resnet152 8,16,32,42 8 $OUT/table1_r152.json > $OUT/table1.log 2>&1
timeout 300 python tools/swap_timeline.py resnet20 32 12 8 8 plan $OUT/r20tl > $OUT/r20tl.log 2>&1
for s in "8232 256 1" "8232 256 1 bwd" "8232 1024 1" "2058 512 1" "16 32 1" "32928 128 1"; do echo "== $s" >> $OUT/bn_trace.txt; timeout 60 python tools/bn_trace.py $s >> $OUT/bn_trace.txt 2>&1; done
