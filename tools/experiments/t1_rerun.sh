OUT=gpurun_out/t1r; mkdir -p $OUT
for i in 1 2; do
  timeout 900 python tools/table1.py resnet152 8,16,32,42 8 $OUT/table1_$i.json > $OUT/table1_$i.log 2>&1
done
