OUT=gpurun_out/${OUT:-r02m}; mkdir -p $OUT
timeout 300 python tools/k1_bench.py > $OUT/k1_bench.jsonl 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
cat $OUT/k1_bench.jsonl; tail -3 $OUT/pytest_gpu.log
