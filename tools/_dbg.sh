timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --csv \
  --log-file gpurun_out/launches_traffic.csv python tools/ncu_step.py resnet152 42 1 > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --profile-from-start off --set full --import-source on -k regex:conv_sm100 -s 60 -c 4 -o gpurun_out/prof_conv_r01 python tools/ncu_step.py resnet152 42 1 > gpurun_out/ncu_full.log 2>&1
timeout 900 ncu --profile-from-start off --set full --import-source on -k regex:bn_fused -s 40 -c 3 -o gpurun_out/prof_bn_r01 python tools/ncu_step.py resnet152 42 1 > gpurun_out/ncu_bn.log 2>&1
timeout 300 python tools/timeline.py resnet152 42 3 gpurun_out/timeline42.json > gpurun_out/timeline42.log 2>&1
