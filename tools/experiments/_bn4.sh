#!/bin/bash
OUT=gpurun_out/bn4; mkdir -p $OUT
timeout 300 python tools/bn_bench.py 42 > $OUT/bn_bench.txt 2>&1
for i in 1 2; do timeout 600 python bench.py --steps 30 --warmup 5 > $OUT/bench_$i.log 2>&1; done
timeout 900 python -m pytest tests/test_layers_gpu.py tests/test_train_step_gpu.py -q -x > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
