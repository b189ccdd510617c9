#!/bin/bash
OUT=gpurun_out/rc2; mkdir -p $OUT
timeout 900 python -m pytest tests/test_layers_gpu.py tests/test_conv_gpu.py -q -x -k "not padd and not kpair" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
timeout 300 python tools/bn_bench.py 42 > $OUT/bn_bench.txt 2>&1
for i in 1 2; do
timeout 600 python bench.py --steps 30 --warmup 5 > $OUT/bench_1_$i.log 2>&1
ACCUDNN_BN_ROWCACHE=0 timeout 600 python bench.py --steps 30 --warmup 5 > $OUT/bench_0_$i.log 2>&1
done
