#!/bin/bash
OUT=gpurun_out/gu; mkdir -p $OUT
for i in 1 2; do timeout 600 python bench.py --steps 30 --warmup 5 > $OUT/bench_$i.log 2>&1; done
ACCUDNN_CONV_BN_STATS=1 timeout 600 python bench.py --steps 30 --warmup 5 > $OUT/bench_stats.log 2>&1
ACCUDNN_CONV_BN_STATS=1 ACCUDNN_BN_STATS_SPLIT=0 timeout 600 python bench.py --steps 30 --warmup 5 > $OUT/bench_stats_coop.log 2>&1
timeout 300 python tools/timeline.py resnet152 42 3 $OUT/timeline.json > $OUT/timeline.log 2>&1
timeout 600 python -m pytest tests/test_swap_executor_gpu.py tests/test_conv_gpu.py -q -k "exposed or stats" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
