OUT=gpurun_out/r02a; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 600 python bench.py > $OUT/bench.log 2>&1; echo "bench rc=$?" >> $OUT/bench.log
timeout 300 python tools/k1_time.py > $OUT/k1_time.log 2>&1
timeout 600 python tools/n0_sweep.py > $OUT/n0_sweep.jsonl 2>&1
ls -la $OUT
