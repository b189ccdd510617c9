timeout 600 python -m pytest tests/test_train_step_gpu.py -q -x > gpurun_out/pytest_gpu.log 2>&1
timeout 600 python bench.py > gpurun_out/bench.log 2>&1
