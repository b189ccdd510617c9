#!/bin/bash
OUT=gpurun_out/epi; mkdir -p $OUT
timeout 900 python -m pytest tests/test_conv_gpu.py -q -x > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
for i in 1 2; do
timeout 600 python bench.py --steps 30 --warmup 5 > $OUT/bench_1_$i.log 2>&1
ACCUDNN_EPI_PIPE=0 timeout 600 python bench.py --steps 30 --warmup 5 > $OUT/bench_0_$i.log 2>&1
done
ACCUDNN_FORCE=256,2,6 timeout 120 python tools/conv_trace.py fwd 42 256 14 14 256 3 1 1 > $OUT/tr_padd.txt 2>&1
ACCUDNN_EPI_PIPE=0 ACCUDNN_FORCE=256,2,6 timeout 120 python tools/conv_trace.py fwd 42 256 14 14 256 3 1 1 > $OUT/tr_padd0.txt 2>&1
