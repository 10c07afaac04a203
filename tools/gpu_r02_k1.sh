OUT=gpurun_out/${OUT:-r02b}; mkdir -p $OUT
timeout 300 python tools/k1_time.py > $OUT/k1_time_team.log 2>&1
CRT_K1_TEAM=0 timeout 300 python tools/k1_time.py > $OUT/k1_time_rolled.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 600 python tools/n0_sweep.py > $OUT/n0_sweep.jsonl 2>&1
timeout 600 python bench.py --no-cpu-baseline --steps 50 > $OUT/bench.log 2>&1
cat $OUT/k1_time_team.log $OUT/k1_time_rolled.log; tail -3 $OUT/pytest_gpu.log
