#!/bin/bash
# pair-add with in-kernel zeroing (no memset node) vs ACCUDNN_PADD_MEMSET=1
OUT=gpurun_out/pnm; mkdir -p $OUT
timeout 900 python -m pytest tests/test_conv_gpu.py -q -x > $OUT/pytest_conv.log 2>&1; echo "rc=$?" >> $OUT/pytest_conv.log
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_conv_gpu.py -q -x -k "padd" > $OUT/memcheck_padd.log 2>&1; echo "rc=$?" >> $OUT/memcheck_padd.log
timeout 900 python -m pytest tests/test_train_step_gpu.py -q -x > $OUT/pytest_step.log 2>&1; echo "rc=$?" >> $OUT/pytest_step.log
for i in 1 2; do
  ACCUDNN_PADD_MEMSET=1 timeout 600 python bench.py --steps 30 --warmup 5 > $OUT/bench_memset_$i.log 2>&1
  timeout 600 python bench.py --steps 30 --warmup 5 > $OUT/bench_inkernel_$i.log 2>&1
done
