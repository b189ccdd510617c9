timeout 900 python bench.py --arch resnet50 --cap-gib 12 --steps 30 > gpurun_out/bench_r50.log 2>&1
