#!/bin/bash
OUT=gpurun_out/bnchk; mkdir -p $OUT
timeout 900 python -m pytest tests/test_layers_gpu.py tests/test_train_step_gpu.py -q -x > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
timeout 300 python tools/bn_bench.py 42 > $OUT/bn_bench.txt 2>&1
for s in "8232 256 1" "8232 256 1 bwd" "8232 1024 1" "2058 512 1" "16 32 1" "32928 128 1"; do echo "== $s" >> $OUT/bn_trace.txt; timeout 60 python tools/bn_trace.py $s >> $OUT/bn_trace.txt 2>&1; done
for i in 1 2; do timeout 600 python bench.py --steps 30 --warmup 5 > $OUT/bench_$i.log 2>&1; done
