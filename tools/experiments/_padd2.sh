#!/bin/bash
OUT=gpurun_out/padd2; mkdir -p $OUT
timeout 900 python -m pytest tests/test_conv_gpu.py -q -x -k "padd or kpair" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
timeout 900 python tools/conv_bench.py 42 $OUT/retune.json retune > $OUT/retune.log 2>&1
