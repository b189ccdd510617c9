#!/bin/bash
# B multicast across clusters of 4 / 8 M-tiles (cm 9 / 10): parity, sweeps, retune A/B
OUT=gpurun_out/mc; mkdir -p $OUT
timeout 900 python -m pytest tests/test_conv_gpu.py -q -x > $OUT/pytest_conv.log 2>&1; echo "rc=$?" >> $OUT/pytest_conv.log
timeout 600 compute-sanitizer --tool memcheck --print-limit 10 python -m pytest tests/test_conv_gpu.py -q -x -k "mc4 or mc8" > $OUT/memcheck_mc.log 2>&1; echo "rc=$?" >> $OUT/memcheck_mc.log
timeout 300 python tools/conv_sweep.py 42 14 14 1024 256 1 1 0 fwd > $OUT/sweep_14_1x1a_fwd.txt 2>&1
timeout 300 python tools/conv_sweep.py 42 14 14 256 1024 1 1 0 dgrad > $OUT/sweep_14_1x1b_dgrad.txt 2>&1
timeout 300 python tools/conv_sweep.py 42 14 14 256 256 3 1 1 fwd > $OUT/sweep_14_3x3_fwd.txt 2>&1
timeout 300 python tools/conv_sweep.py 42 28 28 128 512 1 1 0 fwd > $OUT/sweep_28_1x1_fwd.txt 2>&1
cp profiles/b200/conv_tune.txt /tmp/t_old.txt
ACCUDNN_RETUNE=1 timeout 900 python bench.py --steps 10 --warmup 3 > $OUT/retune.log 2>&1
cp gpurun_out/conv_tune.txt $OUT/conv_tune_new.txt
for i in 1 2; do
  cp /tmp/t_old.txt profiles/b200/conv_tune.txt; timeout 600 python bench.py --steps 30 --warmup 5 > $OUT/bench_old_$i.log 2>&1
  cp $OUT/conv_tune_new.txt profiles/b200/conv_tune.txt; timeout 600 python bench.py --steps 30 --warmup 5 > $OUT/bench_new_$i.log 2>&1
done
cp /tmp/t_old.txt profiles/b200/conv_tune.txt
