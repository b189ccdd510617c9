#!/bin/bash
OUT=gpurun_out/kc2; mkdir -p $OUT
timeout 300 python tools/kc_debug.py > $OUT/kc_debug.txt 2>&1
ACCUDNN_FORCE=256,2,5 timeout 120 python tools/conv_trace.py fwd 42 256 14 14 256 3 1 1 > $OUT/tr_3x3_kc.txt 2>&1
ACCUDNN_FORCE=128,2,5 timeout 120 python tools/conv_trace.py fwd 42 256 14 14 256 3 1 1 > $OUT/tr_3x3_kc128.txt 2>&1
timeout 400 python tools/conv_sweep.py 42 14 14 256 256 3 1 1 fwd > $OUT/sw_3x3_fwd.txt 2>&1
timeout 400 python tools/conv_sweep.py 42 14 14 1024 256 1 1 0 fwd > $OUT/sw_1x1a_fwd.txt 2>&1
