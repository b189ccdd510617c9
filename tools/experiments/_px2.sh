#!/bin/bash
OUT=gpurun_out/px2; mkdir -p $OUT
timeout 900 python -m pytest tests/test_conv_gpu.py -q -k "precise" > $OUT/pytest_conv.log 2>&1; echo "rc=$?" >> $OUT/pytest_conv.log
CONV_MATH=1 timeout 900 python tools/fp32_debug.py resnet152 224 1000 2 > $OUT/dbg_tma.log 2>&1
ACCUDNN_PRECISE_TMA=0 CONV_MATH=1 timeout 900 python tools/fp32_debug.py resnet152 224 1000 2 > $OUT/dbg_cp.log 2>&1
CONV_MATH=1 timeout 900 python tools/fp32_debug.py resnet50 64 8 8 > $OUT/dbg_tma50.log 2>&1
ACCUDNN_PRECISE_TMA=0 CONV_MATH=1 timeout 900 python tools/fp32_debug.py resnet50 64 8 8 > $OUT/dbg_cp50.log 2>&1
