#!/bin/bash
OUT=gpurun_out/bntl; mkdir -p $OUT
timeout 300 python tools/timeline.py resnet152 42 3 $OUT/tl_off.json > $OUT/tl_off.log 2>&1
ACCUDNN_CONV_BN_STATS=3 timeout 300 python tools/timeline.py resnet152 42 3 $OUT/tl_s3.json > $OUT/tl_s3.log 2>&1
