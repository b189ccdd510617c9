timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
timeout 300 python tools/timeline.py resnet152 27 3 gpurun_out/timeline27.json > gpurun_out/timeline27.log 2>&1
timeout 300 python bench.py > gpurun_out/bench.log 2>&1
