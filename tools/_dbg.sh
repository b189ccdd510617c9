timeout 300 python -m pytest tests/test_layers_gpu.py -q -x > gpurun_out/pytest_gpu.log 2>&1
timeout 300 python tools/bn_bench.py 42 > gpurun_out/bn_bench.log 2>&1
python tools/bn_trace.py 8232 256 1 bwd > gpurun_out/bnt3.log 2>&1
timeout 600 python bench.py > gpurun_out/bench.log 2>&1
