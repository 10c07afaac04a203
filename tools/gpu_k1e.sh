OUT=gpurun_out/${OUT:-r02g}; mkdir -p $OUT
timeout 600 ncu --set full --clock-control none --import-source on --warp-sampling-interval 0 -k regex:k1_team -s 5 -c 1 -o $OUT/k1_fc1 python tools/k1_one.py 4608 3072 > $OUT/ncu1.log 2>&1
ls -la $OUT
