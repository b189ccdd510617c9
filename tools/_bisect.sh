#!/bin/bash
OUT=gpurun_out/bisect2; mkdir -p $OUT
ACCUDNN_PRECISE=1 timeout 300 python tools/step_debug.py resnet20 32 12 4 > $OUT/pilot.log 2>&1
cp paper_1901_06773_b200/lib/libaccudnn.so /tmp/main.so
cp tools/alt_lib/libaccudnn_nopilot.so paper_1901_06773_b200/lib/libaccudnn.so
ACCUDNN_PRECISE=1 timeout 300 python tools/step_debug.py resnet20 32 12 4 > $OUT/nopilot.log 2>&1
cp /tmp/main.so paper_1901_06773_b200/lib/libaccudnn.so
