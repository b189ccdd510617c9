#!/bin/bash
# configs 2 / 4 / 5 / 1: runtime tuning graph-timed vs eager-timed (shapes not in the
# committed table are tuned in the first step), and the tuned entries for every config
OUT=gpurun_out/tcfg; mkdir -p $OUT
run() {  # name, extra env, bench args
  local n=$1; shift; local ev=$1; shift
  env $ev timeout 900 python bench.py "$@" > $OUT/$n.log 2>&1
  cp gpurun_out/conv_tune.txt $OUT/$n.tune.txt
}
for i in 1 2; do
  run c4_graph_$i "X=1" --arch resnet152 --cap-gib 12 --steps 30 --warmup 5
  run c4_eager_$i ACCUDNN_TUNE_EAGER=1 --arch resnet152 --cap-gib 12 --steps 30 --warmup 5
  run c2_graph_$i "X=1" --arch resnet50 --cap-gib 12 --steps 30 --warmup 5
  run c2_eager_$i ACCUDNN_TUNE_EAGER=1 --arch resnet50 --cap-gib 12 --steps 30 --warmup 5
done
run c5_graph "X=1" --arch resnet1001 --image 32 --classes 12 --cap-gib 8 --steps 20 --warmup 3
run c1_graph "X=1" --arch resnet20 --image 32 --classes 12 --cap-gib 8 --k 8 --steps 30 --warmup 5
run c3_3x_graph "X=1" --conv-math 3xtf32 --steps 20 --warmup 3
