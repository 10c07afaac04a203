OUT=gpurun_out/${OUT:-r02h}; mkdir -p $OUT
timeout 300 python tools/k1_bench.py > $OUT/k1_bench.jsonl 2>&1
CRT_K1_CPL=1 timeout 300 python tools/k1_bench.py 4608 3072 16 5 4608 3072 16 4 > $OUT/k1_bench_cpl1.jsonl 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
cat $OUT/k1_bench.jsonl $OUT/k1_bench_cpl1.jsonl; tail -15 $OUT/pytest_gpu.log
