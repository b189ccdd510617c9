timeout 900 python -m pytest tests/test_conv_gpu.py -q -x > gpurun_out/pytest_conv.log 2>&1
python tools/conv_trace.py fwd 27 1024 14 14 256 1 1 0 > gpurun_out/trace1.log 2>&1
python tools/conv_trace.py fwd 27 64 56 56 256 1 1 0 > gpurun_out/trace3.log 2>&1
timeout 600 python tools/conv_bench.py 27 gpurun_out/conv_bench.json > gpurun_out/conv_bench.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
timeout 300 python bench.py > gpurun_out/bench.log 2>&1
