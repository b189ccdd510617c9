#!/bin/bash
OUT=gpurun_out/gu3; mkdir -p $OUT
for i in 1 2; do timeout 600 python bench.py --steps 30 --warmup 5 > $OUT/bench_$i.log 2>&1; done
timeout 900 python -m pytest tests/test_swap_executor_gpu.py tests/test_train_step_gpu.py -q > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
timeout 300 python tools/swap_trace.py resnet20 32 12 8 8 plan $OUT/r20 > $OUT/r20.log 2>&1
