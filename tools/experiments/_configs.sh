#!/bin/bash
# every BASELINE single-GPU configuration through bench.py (config 3 is the default line)
OUT=${1:-gpurun_out/configs}; mkdir -p $OUT; rm -f $OUT/configs.jsonl
timeout 900 python bench.py --arch resnet20 --image 32 --classes 12 --cap-gib 8 --k 8 --steps 30 --warmup 5 > $OUT/c1_r20_k8.log 2>&1
timeout 900 python bench.py --arch resnet50 --image 224 --classes 1000 --cap-gib 12 --steps 30 --warmup 5 > $OUT/c2_r50_12g.log 2>&1
timeout 900 python bench.py --arch resnet152 --image 224 --classes 1000 --cap-gib 12 --steps 30 --warmup 5 > $OUT/c4_r152_12g.log 2>&1
timeout 900 python bench.py --arch resnet1001 --image 32 --classes 12 --cap-gib 8 --steps 20 --warmup 3 > $OUT/c5_r1001_8g.log 2>&1
for f in $OUT/*.log; do grep -h '^{' $f | tail -1 >> $OUT/configs.jsonl; done
