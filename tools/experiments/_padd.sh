#!/bin/bash
OUT=gpurun_out/padd; mkdir -p $OUT
timeout 900 python -m pytest tests/test_conv_gpu.py -q -x -k "padd or kpair" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
timeout 400 python tools/conv_sweep.py 42 14 14 256 256 3 1 1 fwd > $OUT/sw_3x3_fwd.txt 2>&1
timeout 400 python tools/conv_sweep.py 42 14 14 1024 256 1 1 0 fwd > $OUT/sw_1x1a_fwd.txt 2>&1
timeout 400 python tools/conv_sweep.py 42 14 14 256 1024 1 1 0 dgrad > $OUT/sw_1x1b_dgrad.txt 2>&1
