#!/bin/bash
OUT=gpurun_out/tr6; mkdir -p $OUT
ACCUDNN_FORCE=256,2,6 timeout 120 python tools/conv_trace.py fwd 42 256 14 14 256 3 1 1 > $OUT/tr_3x3_padd.txt 2>&1
ACCUDNN_FORCE=256,2,1 timeout 120 python tools/conv_trace.py fwd 42 256 14 14 256 3 1 1 > $OUT/tr_3x3_ws.txt 2>&1
timeout 300 ncu --clock-control none --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second,smsp__cycles_active.avg --csv --log-file $OUT/ncu_padd.csv python tools/conv_one.py 42 14 14 256 256 3 1 1 fwd 256,2,6 > /dev/null 2>&1
timeout 300 ncu --clock-control none --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second,smsp__cycles_active.avg --csv --log-file $OUT/ncu_tuned128.csv python tools/conv_one.py 42 14 14 256 256 3 1 1 fwd 128,1,1 > /dev/null 2>&1
