#!/bin/bash
OUT=gpurun_out/cv1; mkdir -p $OUT
for s in "8232 256 1" "8232 256 1 bwd" "2058 512 1" "32928 128 1"; do echo "== $s" >> $OUT/bn_trace.txt; timeout 60 python tools/bn_trace.py $s >> $OUT/bn_trace.txt 2>&1; done
timeout 300 python tools/conv_sweep.py 42 14 14 256 256 3 1 1 fwd > $OUT/sw_3x3_fwd.txt 2>&1
timeout 300 python tools/conv_sweep.py 42 14 14 256 256 3 1 1 dgrad > $OUT/sw_3x3_dgrad.txt 2>&1
timeout 300 python tools/conv_sweep.py 42 14 14 1024 256 1 1 0 fwd > $OUT/sw_1x1a_fwd.txt 2>&1
timeout 300 python tools/conv_sweep.py 42 14 14 256 1024 1 1 0 dgrad > $OUT/sw_1x1b_dgrad.txt 2>&1
