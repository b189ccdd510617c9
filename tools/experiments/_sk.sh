#!/bin/bash
OUT=gpurun_out/sk; mkdir -p $OUT
timeout 900 python -m pytest tests/test_conv_gpu.py -q -x > $OUT/conv_tests.log 2>&1; echo "rc=$?" >> $OUT/conv_tests.log
timeout 600 python tools/conv_bench.py 42 $OUT/bench_table.json table > $OUT/bench_table.log 2>&1
timeout 600 python tools/conv_bench.py 42 $OUT/bench_sk.json sk > $OUT/bench_sk.log 2>&1
timeout 900 python tools/conv_bench.py 42 $OUT/bench_retune.json retune > $OUT/bench_retune.log 2>&1
