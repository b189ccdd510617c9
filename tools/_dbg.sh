timeout 600 python -m pytest tests/test_conv_gpu.py -q -x > gpurun_out/pytest_conv.log 2>&1
ACCUDNN_FORCE=128,1,1 python tools/conv_trace.py fwd 42 256 14 14 1024 1 1 0 > gpurun_out/t_a.log 2>&1
ACCUDNN_FORCE=128,1,3 python tools/conv_trace.py fwd 42 256 14 14 1024 1 1 0 > gpurun_out/t_b.log 2>&1
ACCUDNN_FORCE=256,1,3 python tools/conv_trace.py fwd 42 256 14 14 1024 1 1 0 > gpurun_out/t_c.log 2>&1
ACCUDNN_FORCE=64,1,3 python tools/conv_trace.py fwd 42 1024 14 14 256 1 1 0 > gpurun_out/t_d.log 2>&1
ACCUDNN_FORCE=128,1,1 python tools/conv_trace.py fwd 42 1024 14 14 256 1 1 0 > gpurun_out/t_e.log 2>&1
