#!/bin/bash
# One gpurun call: GPU tests, smoke, bench line, ncu launch list + full capture
# of the top conv kernel.  Outputs under gpurun_out/.
set -x
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
nproc > $OUT/nproc.txt; lscpu > $OUT/lscpu.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench.log 2>&1; echo "bench rc=$?" >> $OUT/bench.log
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_ref.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv \
  --log-file $OUT/launches.csv python tools/ncu_step.py resnet152 ${KSTAR:-27} 0 > $OUT/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:conv_tma -s 40 -c 3 \
  -o $OUT/prof_conv python tools/ncu_step.py resnet152 ${KSTAR:-27} 0 > $OUT/ncu_full.log 2>&1
ls -la $OUT
