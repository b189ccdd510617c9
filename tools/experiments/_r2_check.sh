#!/bin/bash
OUT=gpurun_out/r2check
mkdir -p $OUT
timeout 1200 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 900 python bench.py --steps 20 --warmup 3 > $OUT/bench.log 2>&1; echo "bench rc=$?" >> $OUT/bench.log
timeout 900 python bench.py --impl reference --steps 20 --warmup 3 > $OUT/bench_ref.log 2>&1; echo "ref rc=$?" >> $OUT/bench_ref.log
