OUT=gpurun_out/${OUT:-r02n}; mkdir -p $OUT
for R in _ab/base . _ab/base .; do echo "== $R"; CRT_ROOT=$R timeout 300 python tools/k1_bench.py 4608 3072 16 5 4608 12288 16 5 4608 15360 16 5 4608 3072 4 5; done > $OUT/ab.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
cat $OUT/ab.txt; tail -2 $OUT/pytest_gpu.log
