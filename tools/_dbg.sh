timeout 600 ncu --set full --import-source on -k regex:bn_fused -s 2 -c 1 -o gpurun_out/prof_bn1 python tools/_bn_one.py 1323 512 > gpurun_out/ncu_bn1.log 2>&1
timeout 600 ncu --set full --import-source on -k regex:bn_fused -s 2 -c 1 -o gpurun_out/prof_bn2 python tools/_bn_one.py 5292 256 > gpurun_out/ncu_bn2.log 2>&1
