#!/bin/bash
# compute-sanitizer over this round's kernels (final code); outputs under gpurun_out/san
OUT=gpurun_out/san; mkdir -p $OUT
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_conv_gpu.py -q -x -k "kpair and 14 or precise or padd" > $OUT/memcheck_conv.log 2>&1; echo "rc=$?" >> $OUT/memcheck_conv.log
timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_layers_gpu.py -q -x -k "batchnorm or bn" > $OUT/memcheck_bn.log 2>&1; echo "rc=$?" >> $OUT/memcheck_bn.log
timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_swap_executor_gpu.py -q -x -k "order or documents" > $OUT/memcheck_swap.log 2>&1; echo "rc=$?" >> $OUT/memcheck_swap.log
timeout 1200 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_layers_gpu.py -q -x -k "batchnorm or bn" > $OUT/racecheck_bn.log 2>&1; echo "rc=$?" >> $OUT/racecheck_bn.log
timeout 1200 compute-sanitizer --tool synccheck --print-limit 20 python -m pytest tests/test_layers_gpu.py -q -x -k "batchnorm or bn" > $OUT/synccheck_bn.log 2>&1; echo "rc=$?" >> $OUT/synccheck_bn.log
timeout 1200 compute-sanitizer --tool synccheck --print-limit 20 python -m pytest tests/test_conv_gpu.py -q -x -k "kpair and 14" > $OUT/synccheck_kc.log 2>&1; echo "rc=$?" >> $OUT/synccheck_kc.log
for f in $OUT/*.log; do echo "== $f"; tail -n 4 "$f"; done
