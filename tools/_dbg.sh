timeout 600 python -m pytest tests/test_conv_gpu.py -x -q > gpurun_out/pytest_conv.log 2>&1
timeout 600 python tools/conv_bench.py 27 gpurun_out/conv_bench.json > gpurun_out/conv_bench.log 2>&1
timeout 600 python bench.py > gpurun_out/bench.log 2>&1
