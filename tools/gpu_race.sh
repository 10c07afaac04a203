OUT=gpurun_out/${OUT:-r02t}; mkdir -p $OUT
SAN_TP=0 timeout 1500 /usr/local/cuda/bin/compute-sanitizer --tool racecheck --print-limit 20 python tools/sanitize_workload.py > $OUT/racecheck.log 2>&1; echo "rc=$?" >> $OUT/racecheck.log
grep -E "RACECHECK SUMMARY|sanitize workload|rc=|Read access at" $OUT/racecheck.log | sort | uniq -c | head
timeout 600 python -m pytest tests/test_k3_v3.py tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -1
