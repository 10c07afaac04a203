OUT=gpurun_out/${OUT:-r02d}; mkdir -p $OUT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k1_team -s 5 -c 1 -o $OUT/k1_fc1 python tools/k1_one.py 4608 3072 > $OUT/ncu1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k1_team -s 5 -c 1 -o $OUT/k1_fc2 python tools/k1_one.py 4608 12288 > $OUT/ncu2.log 2>&1
tail -2 $OUT/ncu1.log $OUT/ncu2.log; ls -la $OUT
