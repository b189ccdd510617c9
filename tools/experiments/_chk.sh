#!/bin/bash
# quick GPU check: selected test files, bench x2, optional extra command
OUT=gpurun_out/chk; mkdir -p $OUT
timeout 900 python -m pytest ${TESTS:-tests/test_conv_gpu.py tests/test_layers_gpu.py tests/test_train_step_gpu.py} -q -x > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest.log
for i in 1 2; do timeout 600 python bench.py --steps 30 --warmup 5 > $OUT/bench_$i.log 2>&1; done
if [ -n "$EXTRA" ]; then bash -c "$EXTRA" > $OUT/extra.log 2>&1; fi
tail -2 $OUT/pytest.log; grep -h -o '"value": [0-9.]*, "unit": "images/s", "n_gpus"' $OUT/bench_*.log
