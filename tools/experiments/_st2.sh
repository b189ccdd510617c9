#!/bin/bash
OUT=gpurun_out/st2; mkdir -p $OUT
for i in 1 2; do
timeout 600 python bench.py --steps 30 --warmup 5 > $OUT/bench_0_$i.log 2>&1
ACCUDNN_CONV_BN_STATS=2 timeout 600 python bench.py --steps 30 --warmup 5 > $OUT/bench_2_$i.log 2>&1
done
ACCUDNN_CONV_BN_STATS=2 timeout 900 python -m pytest tests/test_train_step_gpu.py -q -x -k "not r152" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
