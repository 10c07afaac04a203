# compute-sanitizer over tools/sanitize_workload.py (every kernel family).
# The default process runs K3 v4 for W4A4; a second memcheck pass runs the
# same workload with CRT_K3_V3=1 (the v3 kernel).  OUT=<name> bash tools/gpu_sanitize.sh
OUT=gpurun_out/${OUT:-r02s}; mkdir -p $OUT
CS=/usr/local/cuda/bin/compute-sanitizer
for T in memcheck synccheck racecheck; do
  SAN_TP=$([ $T = memcheck ] && echo 1 || echo 0) timeout 1500 $CS --tool $T --print-limit 20 --target-processes all python tools/sanitize_workload.py > $OUT/$T.log 2>&1
  echo "$T rc=$?" >> $OUT/$T.log
  echo "== $T"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|sanitize workload|rc=|Error|Hazard" $OUT/$T.log | head -8
done
CRT_K3_V3=1 timeout 1500 $CS --tool memcheck --print-limit 20 --target-processes all python tools/sanitize_workload.py > $OUT/memcheck_v3.log 2>&1
echo "memcheck_v3 rc=$?" >> $OUT/memcheck_v3.log
echo "== memcheck (CRT_K3_V3=1)"; grep -E "ERROR SUMMARY|sanitize workload|rc=" $OUT/memcheck_v3.log | head -4
