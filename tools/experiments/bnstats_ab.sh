#!/bin/bash
# conv-epilogue BN statistics on the large layers only (ACCUDNN_CONV_BN_STATS=3) vs off
OUT=gpurun_out/bnst; mkdir -p $OUT
timeout 900 python -m pytest tests/test_train_step_gpu.py -q -x -k "graph_step_matches_eager or tf32_mode" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
ACCUDNN_CONV_BN_STATS=3 timeout 900 python -m pytest tests/test_train_step_gpu.py -q -x -k "graph_step_matches_eager or tf32_mode" > $OUT/pytest_s3.log 2>&1; echo "rc=$?" >> $OUT/pytest_s3.log
for i in 1 2; do
  timeout 600 python bench.py --steps 30 --warmup 5 > $OUT/bench_off_$i.log 2>&1
  ACCUDNN_CONV_BN_STATS=3 timeout 600 python bench.py --steps 30 --warmup 5 > $OUT/bench_s3_$i.log 2>&1
  ACCUDNN_CONV_BN_STATS=3 ACCUDNN_BN_STATS_SPLIT=1 timeout 600 python bench.py --steps 30 --warmup 5 > $OUT/bench_s3split_$i.log 2>&1
done
