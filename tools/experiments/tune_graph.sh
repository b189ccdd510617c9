#!/bin/bash
# conv tuner timing candidates as CUDA graphs: retune, then A/B against the
# committed table and the eager-timed retune
OUT=gpurun_out/tgraph; mkdir -p $OUT
timeout 900 python -m pytest tests/test_conv_gpu.py -q -x -k "tune or padd or streamk" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
cp profiles/b200/conv_tune.txt /tmp/t_old.txt
ACCUDNN_RETUNE=1 timeout 900 python bench.py --steps 10 --warmup 3 > $OUT/retune.log 2>&1
cp gpurun_out/conv_tune.txt $OUT/conv_tune_graph.txt
for i in 1 2; do
  cp /tmp/t_old.txt profiles/b200/conv_tune.txt; timeout 600 python bench.py --steps 30 --warmup 5 > $OUT/bench_old_$i.log 2>&1
  cp _ab/tune_eager_retune.txt profiles/b200/conv_tune.txt; timeout 600 python bench.py --steps 30 --warmup 5 > $OUT/bench_eager_$i.log 2>&1
  cp $OUT/conv_tune_graph.txt profiles/b200/conv_tune.txt; timeout 600 python bench.py --steps 30 --warmup 5 > $OUT/bench_graph_$i.log 2>&1
done
cp /tmp/t_old.txt profiles/b200/conv_tune.txt
cp profiles/b200/conv_tune.txt /tmp/t_old.txt
timeout 300 python tools/conv_sweep.py 42 14 14 256 256 3 1 1 fwd > $OUT/sweep_14_3x3_fwd.txt 2>&1
