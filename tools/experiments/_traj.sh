#!/bin/bash
OUT=gpurun_out/traj; mkdir -p $OUT
timeout 900 python -m pytest tests/test_train_step_gpu.py -q -k "trajectory" > $OUT/t_default.log 2>&1
ACCUDNN_TUNE_VARIANTS=4 timeout 900 python -m pytest tests/test_train_step_gpu.py -q -k "trajectory" > $OUT/t_v4.log 2>&1
ACCUDNN_TUNE_VARIANTS=5 timeout 900 python -m pytest tests/test_train_step_gpu.py -q -k "trajectory" > $OUT/t_v5.log 2>&1
tail -1 $OUT/*.log
