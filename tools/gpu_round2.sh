#!/bin/bash
# One gpurun call producing round-2 evidence under gpurun_out/r02/.
OUT=gpurun_out/r02
mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1; nproc > $OUT/nproc.txt; lscpu > $OUT/lscpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench.log 2>&1; echo "bench rc=$?" >> $OUT/bench.log
timeout 900 python bench.py --conv-math 3xtf32 > $OUT/bench_3xtf32.log 2>&1; echo "rc=$?" >> $OUT/bench_3xtf32.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/bench_ref.log 2>&1; echo "rc=$?" >> $OUT/bench_ref.log
timeout 900 ncu --profile-from-start off --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --csv \
  --log-file $OUT/launches_k42.csv python tools/ncu_step.py resnet152 42 1 > $OUT/ncu_launch.log 2>&1
python tools/summarize_launches.py $OUT/launches_k42.csv $OUT/launch_summary_k42.json > $OUT/launch_summary_k42.md 2>&1
timeout 900 ncu --profile-from-start off --clock-control none --set full --import-source on -k regex:conv_sm100 -s 60 -c 4 -o $OUT/prof_conv python tools/ncu_step.py resnet152 42 1 > $OUT/ncu_full.log 2>&1
timeout 900 ncu --profile-from-start off --clock-control none --set full --import-source on -k regex:bn_fused -s 40 -c 3 -o $OUT/prof_bn python tools/ncu_step.py resnet152 42 1 > $OUT/ncu_bn.log 2>&1
timeout 300 python tools/timeline.py resnet152 42 3 $OUT/timeline_k42.json > $OUT/timeline_k42.log 2>&1
timeout 900 python tools/swap_stress.py $OUT/swap_stress.json > $OUT/swap_stress.log 2>&1
timeout 600 python tools/copy_bench.py $OUT/copy_bench.json > $OUT/copy_bench.log 2>&1
timeout 900 python tools/table1.py resnet152 8,16,32,42 8 $OUT/table1_r152.json > $OUT/table1.log 2>&1
timeout 600 python tools/conv_bench.py 42 $OUT/conv_bench_k42.json > $OUT/conv_bench.log 2>&1
timeout 300 python tools/bn_bench.py 42 > $OUT/bn_bench_k42.txt 2>&1
ls -la $OUT
