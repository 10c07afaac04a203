OUT=gpurun_out/${OUT:-r02f}; mkdir -p $OUT
for R in . _ab/r72 _ab/r64; do echo "== $R"; CRT_ROOT=$R timeout 300 python tools/k1_bench.py 4608 3072 16 5 4608 12288 16 5 4608 3072 64 5 4608 3072 256 5 4608 15360 16 5 4096 3072 16 5; done > $OUT/k1_regs.txt 2>&1
timeout 120 python tools/k1_trace.py 4608 3072 > $OUT/trace_fc1.txt 2>&1
cat $OUT/k1_regs.txt; head -20 $OUT/trace_fc1.txt
