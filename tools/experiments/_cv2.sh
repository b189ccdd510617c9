#!/bin/bash
OUT=gpurun_out/cv2; mkdir -p $OUT
timeout 120 python tools/conv_trace.py fwd 42 256 14 14 256 3 1 1 > $OUT/tr_3x3_fwd_tuned.txt 2>&1
ACCUDNN_FORCE=256,2,1 timeout 120 python tools/conv_trace.py fwd 42 256 14 14 256 3 1 1 > $OUT/tr_3x3_fwd_256_2.txt 2>&1
ACCUDNN_FORCE=128,1,4 timeout 120 python tools/conv_trace.py fwd 42 256 14 14 256 3 1 1 > $OUT/tr_3x3_fwd_pair.txt 2>&1
timeout 120 python tools/conv_trace.py fwd 42 1024 14 14 256 1 1 0 > $OUT/tr_1x1_fwd_tuned.txt 2>&1
timeout 900 python -m pytest tests/test_layers_gpu.py tests/test_train_step_gpu.py -q -x > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
timeout 300 python tools/bn_bench.py 42 > $OUT/bn_bench.txt 2>&1
for i in 1 2; do timeout 600 python bench.py --steps 30 --warmup 5 > $OUT/bench_$i.log 2>&1; done
