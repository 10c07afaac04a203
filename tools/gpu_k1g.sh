OUT=gpurun_out/${OUT:-r02i}; mkdir -p $OUT
timeout 300 python tools/k1_bench.py > $OUT/k1_bench.jsonl 2>&1
CRT_K1_CPL=2 timeout 300 python tools/k1_bench.py 4608 3072 16 5 4608 12288 16 5 > $OUT/k1_bench_cpl2.jsonl 2>&1
CRT_ROOT=_ab/tr timeout 120 python tools/k1_trace.py 4608 3072 > $OUT/trace_fc1.txt 2>&1
CRT_ROOT=_ab/tr timeout 120 python tools/k1_trace.py 4608 12288 > $OUT/trace_fc2.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
cat $OUT/k1_bench.jsonl $OUT/k1_bench_cpl2.jsonl; head -12 $OUT/trace_fc1.txt; head -12 $OUT/trace_fc2.txt; tail -3 $OUT/pytest_gpu.log
