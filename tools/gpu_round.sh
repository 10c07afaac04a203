#!/bin/bash
# One gpurun call: GPU parity tests, smoke, bench, ncu launch list + full captures.
# usage: gpurun -- bash tools/gpu_round.sh [tag]
TAG=${1:-r01}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 600 python bench.py > $OUT/bench.log 2>&1; echo "bench rc=$?" >> $OUT/bench.log
timeout 600 python bench.py --path v2 --no-cpu-baseline --no-e2e > $OUT/bench_v2.log 2>&1
timeout 900 python tools/flux_stack.py > $OUT/flux_stack.jsonl 2>&1
timeout 300 python tools/k1_time.py > $OUT/k1_time.log 2>&1
timeout 300 python tools/n0_sweep.py > $OUT/n0_sweep.jsonl 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
  python bench.py --steps 2 --warmup 3 --profile > $OUT/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k3_v3 -s 2 -c 1 \
  -o $OUT/k3 python bench.py --steps 2 --warmup 3 --profile > $OUT/ncu_k3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k1_(fast|rolled)" -s 4 -c 2 \
  -o $OUT/k1 python bench.py --steps 2 --warmup 3 --profile > $OUT/ncu_k1.log 2>&1
ls -la $OUT
