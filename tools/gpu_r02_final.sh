# Round-2 evidence run: GPU tests, smoke, default bench line, FLUX stack,
# ncu launch list of the bench, ncu --set full of K3 (fc1) and K1 (fc1).
# OUT=<name> bash tools/gpu_r02_final.sh
OUT=gpurun_out/${OUT:-r02z}; mkdir -p $OUT
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench.log 2>&1; echo "bench rc=$?" >> $OUT/bench.log
timeout 900 python tools/flux_stack.py > $OUT/flux_stack.jsonl 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv python bench.py --steps 2 --warmup 3 --profile > $OUT/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k3_v4 -s 2 -c 1 -o $OUT/k3 python tools/k3_one.py 4608 3072 12288 3 > $OUT/ncu_k3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k1_team -s 5 -c 1 -o $OUT/k1 python tools/k1_one.py 4608 3072 > $OUT/ncu_k1.log 2>&1
tail -2 $OUT/pytest_gpu.log $OUT/smoke.log; tail -3 $OUT/bench.log; ls -la $OUT
