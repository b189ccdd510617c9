#!/bin/bash
# weight-gradient stream CTA cap (ACCUDNN_SIDE_CTAS) A/B
OUT=gpurun_out/sidec; mkdir -p $OUT
for i in 1 2; do
  for n in 0 111 74 37; do
    ACCUDNN_SIDE_CTAS=$n timeout 600 python bench.py --steps 30 --warmup 5 > $OUT/bench_s${n}_$i.log 2>&1
  done
done
