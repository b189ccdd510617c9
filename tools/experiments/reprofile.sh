OUT=gpurun_out/reprof; mkdir -p $OUT
timeout 2400 python tools/profile_b200.py --archs resnet152,resnet50,resnet20,resnet1001 > $OUT/profile.log 2>&1; echo "rc=$?" >> $OUT/profile.log
cp profiles/b200/*.csv profiles/b200/host_link.json $OUT/
timeout 900 python tools/table1.py resnet152 8,16,32,42 8 $OUT/table1_r152.json > $OUT/table1.log 2>&1
