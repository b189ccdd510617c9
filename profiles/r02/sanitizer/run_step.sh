#!/bin/bash
# compute-sanitizer memcheck over whole training steps (ResNet-20/50 cases of the step tests, the swap executor)
OUT=gpurun_out/san2; mkdir -p $OUT
timeout 2700 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_train_step_gpu.py -q -x -k "not r152" > $OUT/memcheck_step.log 2>&1; echo "rc=$?" >> $OUT/memcheck_step.log
timeout 1800 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_swap_executor_gpu.py -q -x -k "order or documents" > $OUT/memcheck_swap_all.log 2>&1; echo "rc=$?" >> $OUT/memcheck_swap_all.log
for f in $OUT/*.log; do echo "== $f"; tail -n 4 "$f"; done
