#!/bin/bash
OUT=gpurun_out/ab2; mkdir -p $OUT
B="python bench.py --steps 30 --warmup 5"
for i in 1 2; do
for c in f563dd7 f8af7b6 7d05672 r1; do
(cd _ab/$c && timeout 600 $B > ../../$OUT/${c}_$i.log 2>&1)
done
done
