#!/bin/bash
OUT=gpurun_out/sw3; mkdir -p $OUT
timeout 600 python -m pytest tests/test_conv_gpu.py tests/test_swap_executor_gpu.py -q > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
timeout 300 python tools/swap_timeline.py resnet20 32 12 8 8 plan $OUT/r20tl > $OUT/r20tl.log 2>&1
