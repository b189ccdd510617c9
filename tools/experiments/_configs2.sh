#!/bin/bash
OUT=gpurun_out/configs2; mkdir -p $OUT
timeout 900 python bench.py --arch resnet20 --image 32 --classes 12 --cap-gib 8 --k 8 --steps 30 --warmup 5 > $OUT/c1_r20_k8.log 2>&1
timeout 1500 python bench.py --arch resnet1001 --image 32 --classes 12 --cap-gib 8 --steps 20 --warmup 3 > $OUT/c5_r1001_8g.log 2>&1
