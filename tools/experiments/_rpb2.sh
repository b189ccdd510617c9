#!/bin/bash
OUT=gpurun_out/rpb2; mkdir -p $OUT
timeout 300 python tools/bn_bench.py 42 > $OUT/bn_bench.txt 2>&1
for i in 1 2; do timeout 600 python bench.py --steps 30 --warmup 5 > $OUT/bench_$i.log 2>&1; done
timeout 1500 python -m pytest tests -m gpu -q > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
