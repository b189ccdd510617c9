#!/bin/bash
OUT=gpurun_out/rw; mkdir -p $OUT
timeout 900 python -m pytest tests/test_conv_gpu.py -q -x > $OUT/pytest_conv.log 2>&1; echo "rc=$?" >> $OUT/pytest_conv.log
for i in 1 2; do timeout 600 python bench.py --steps 30 --warmup 5 > $OUT/bench_$i.log 2>&1; done
timeout 600 python tools/conv_bench.py 42 $OUT/conv_bench.json > $OUT/conv_bench.log 2>&1
