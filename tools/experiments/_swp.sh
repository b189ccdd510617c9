#!/bin/bash
OUT=gpurun_out/swp; mkdir -p $OUT
timeout 300 python tools/swap_trace.py resnet20 32 12 8 8 plan $OUT/r20_k > $OUT/r20_k.log 2>&1
ACCUDNN_KCOPY_D2H=0 ACCUDNN_KCOPY_H2D=0 timeout 300 python tools/swap_trace.py resnet20 32 12 8 8 plan $OUT/r20_e > $OUT/r20_e.log 2>&1
ACCUDNN_KCOPY_D2H=100000000 ACCUDNN_KCOPY_H2D=100000000 timeout 300 python tools/swap_trace.py resnet20 32 12 8 8 plan $OUT/r20_kall > $OUT/r20_kall.log 2>&1
timeout 300 python tools/swap_timeline.py resnet20 32 12 8 8 plan $OUT/r20tl > $OUT/r20tl.log 2>&1
timeout 900 python -m pytest tests/test_swap_executor_gpu.py tests/test_train_step_gpu.py -q > $OUT/pytest.log 2>&1
timeout 900 python tools/swap_stress.py $OUT/swap_stress.json > $OUT/stress.log 2>&1
grep exposed_frac_graph $OUT/*.log
timeout 300 python tools/fp32_debug.py resnet50 64 8 8 > $OUT/fp32dbg.log 2>&1
