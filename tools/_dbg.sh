timeout 900 python -m pytest tests/test_layers_gpu.py tests/test_train_step_gpu.py -q > gpurun_out/pytest_gpu.log 2>&1
timeout 600 python bench.py > gpurun_out/bench.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv \
  --log-file gpurun_out/launches.csv python tools/ncu_step.py resnet152 27 0 > gpurun_out/ncu_launch.log 2>&1
