timeout 600 python -m pytest tests/test_cli.py -q -m gpu > gpurun_out/pytest_cli.log 2>&1
timeout 900 python tools/table1.py resnet152 8,16,32,42 8 gpurun_out/table1_r152.json > gpurun_out/table1.log 2>&1
