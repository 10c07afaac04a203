OUT=gpurun_out/${OUT:-r02o}; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 900 python tools/flux_stack.py --steps 3 > $OUT/flux_stack.jsonl 2>&1
tail -5 $OUT/pytest_gpu.log; cat $OUT/flux_stack.jsonl
