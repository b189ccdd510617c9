#!/bin/bash
# One gpurun call producing the round's evidence: GPU tests, smoke, bench
# line (+ reference arm), ncu launch list with DRAM traffic, ncu --set full of
# conv and BN launches, CUPTI timeline.  Outputs under gpurun_out/.
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
nproc > $OUT/nproc.txt
timeout 900 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench.log 2>&1; echo "bench rc=$?" >> $OUT/bench.log
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_ref.log 2>&1
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --csv \
  --log-file $OUT/launches_traffic.csv python tools/ncu_step.py resnet152 ${KSTAR:-42} 1 > $OUT/ncu_launch.log 2>&1
timeout 900 ncu --profile-from-start off --set full --import-source on -k regex:conv_sm100 -s 60 -c 4 -o $OUT/prof_conv_r01 python tools/ncu_step.py resnet152 ${KSTAR:-42} 1 > $OUT/ncu_full.log 2>&1
timeout 900 ncu --profile-from-start off --set full --import-source on -k regex:bn_fused -s 40 -c 3 -o $OUT/prof_bn_r01 python tools/ncu_step.py resnet152 ${KSTAR:-42} 1 > $OUT/ncu_bn.log 2>&1
timeout 300 python tools/timeline.py resnet152 ${KSTAR:-42} 3 $OUT/timeline42.json > $OUT/timeline42.log 2>&1
timeout 600 python tools/conv_bench.py ${KSTAR:-42} $OUT/conv_bench42.json > $OUT/conv_bench42.log 2>&1
timeout 300 python tools/bn_bench.py ${KSTAR:-42} > $OUT/bn_bench.log 2>&1
ls -la $OUT
