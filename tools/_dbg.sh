ACCUDNN_FORCE=128,1,1 python tools/conv_trace.py fwd 42 1024 14 14 256 1 1 0 > gpurun_out/t_a.log 2>&1
ACCUDNN_FORCE=128,1,2 python tools/conv_trace.py fwd 42 1024 14 14 256 1 1 0 > gpurun_out/t_b.log 2>&1
ACCUDNN_FORCE=256,1,2 python tools/conv_trace.py fwd 42 1024 14 14 256 1 1 0 > gpurun_out/t_c.log 2>&1
ACCUDNN_FORCE=128,1,1 python tools/conv_trace.py fwd 42 256 14 14 256 3 1 1 > gpurun_out/t_d.log 2>&1
ACCUDNN_FORCE=128,1,2 python tools/conv_trace.py fwd 42 256 14 14 256 3 1 1 > gpurun_out/t_e.log 2>&1
ACCUDNN_FORCE=256,2,2 python tools/conv_trace.py fwd 42 256 14 14 256 3 1 1 > gpurun_out/t_f.log 2>&1
