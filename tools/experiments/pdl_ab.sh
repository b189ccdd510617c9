# Re-profiled documents: GPU suite, bench, config sweep; PDL A/B on the bench step.
OUT=gpurun_out/pdl; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
for i in 1 2; do
  for p in 0 1; do
    ACCUDNN_PDL=$p timeout 600 python bench.py > $OUT/bench_pdl${p}_$i.log 2>&1
  done
done
timeout 900 python tools/swap_stress.py $OUT/swap_stress.json > $OUT/swap_stress.log 2>&1
