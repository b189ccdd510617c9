timeout 600 python -m pytest tests/test_layers_gpu.py -q -x > gpurun_out/pytest_gpu.log 2>&1
timeout 300 python tools/timeline.py resnet152 42 3 gpurun_out/timeline42.json > gpurun_out/timeline42.log 2>&1
