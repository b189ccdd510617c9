#!/bin/bash
OUT=gpurun_out/px; mkdir -p $OUT
timeout 900 python -m pytest tests/test_conv_gpu.py -q -x -k "precise" > $OUT/pytest_conv.log 2>&1; echo "rc=$?" >> $OUT/pytest_conv.log
timeout 900 python -m pytest tests/test_train_step_gpu.py -q -x > $OUT/pytest_step.log 2>&1; echo "rc=$?" >> $OUT/pytest_step.log
timeout 900 python bench.py --conv-math 3xtf32 --steps 10 --warmup 3 > $OUT/bench_3x.log 2>&1
tail -2 $OUT/pytest_conv.log $OUT/pytest_step.log
