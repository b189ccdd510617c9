timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 600 python tools/conv_bench.py 27 gpurun_out/conv_bench.json > gpurun_out/conv_bench.log 2>&1
