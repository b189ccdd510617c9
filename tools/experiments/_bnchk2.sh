#!/bin/bash
OUT=gpurun_out/bnchk2; mkdir -p $OUT
timeout 300 python tools/bn_bench.py 42 > $OUT/bn_bench.txt 2>&1
ACCUDNN_BN_CLUSTER=1 timeout 300 python tools/bn_bench.py 42 > $OUT/bn_bench_cl1.txt 2>&1
ACCUDNN_BN_CLUSTER=0 timeout 300 python tools/bn_bench.py 42 > $OUT/bn_bench_cl0.txt 2>&1
for s in "8232 256 1" "2058 512 1" "8232 1024 1" "32928 128 1"; do echo "== $s" >> $OUT/bn_trace.txt; timeout 60 python tools/bn_trace.py $s >> $OUT/bn_trace.txt 2>&1; done
TABLE1_MODES=naive ACCUDNN_KCOPY_D2H=0 ACCUDNN_KCOPY_H2D=0 timeout 600 python tools/table1.py resnet152 16 8 $OUT/t1_nokc.json > $OUT/t1_nokc.log 2>&1
TABLE1_MODES=naive timeout 600 python tools/table1.py resnet152 16 8 $OUT/t1_kc.json > $OUT/t1_kc.log 2>&1
timeout 600 python tools/swap_trace.py resnet152 224 1000 16 8 naive $OUT/n16 > $OUT/n16.log 2>&1
