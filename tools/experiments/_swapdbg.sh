#!/bin/bash
OUT=gpurun_out/swapdbg; mkdir -p $OUT
timeout 300 python -m pytest tests/test_train_step_gpu.py -q -k "fp32_mode" > $OUT/fp32.log 2>&1
timeout 300 python -m pytest tests/test_layers_gpu.py -q -k "batchnorm" > $OUT/bn.log 2>&1
timeout 300 python tools/swap_trace.py resnet20 32 12 8 8 plan $OUT/r20 > $OUT/r20.log 2>&1
ACCUDNN_PREFETCH=lookahead timeout 300 python tools/swap_trace.py resnet20 32 12 8 8 plan $OUT/r20_la > $OUT/r20_la.log 2>&1
timeout 300 python tools/swap_trace.py resnet50 64 8 16 8 every3 $OUT/r50 > $OUT/r50.log 2>&1
