timeout 900 python -m pytest tests/test_train_step_gpu.py -q -x > gpurun_out/pytest_gpu.log 2>&1
timeout 600 python tools/swap_bench.py 8 gpurun_out/swap_bench_k8.json > gpurun_out/swap_bench.log 2>&1
timeout 600 python tools/swap_bench.py 48 gpurun_out/swap_bench_k48.json > gpurun_out/swap_bench48.log 2>&1
