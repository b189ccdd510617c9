#!/bin/bash
OUT=gpurun_out/swp2; mkdir -p $OUT
timeout 600 python tools/copy_bench.py $OUT/copy_bench.json > $OUT/copy.log 2>&1
timeout 1500 python -m pytest tests/test_swap_executor_gpu.py tests/test_train_step_gpu.py -q > $OUT/pytest.log 2>&1
timeout 300 python tools/swap_trace.py resnet20 32 12 8 8 plan $OUT/r20_k > $OUT/r20_k.log 2>&1
timeout 900 python tools/fp32_debug.py resnet152 224 1000 2 > $OUT/fp32dbg152.log 2>&1
