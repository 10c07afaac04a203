OUT=gpurun_out/${OUT:-r02s}; mkdir -p $OUT
CS=/usr/local/cuda/bin/compute-sanitizer
for T in memcheck synccheck racecheck; do
  SAN_TP=$([ $T = memcheck ] && echo 1 || echo 0) timeout 1500 $CS --tool $T --print-limit 20 --target-processes all python tools/sanitize_workload.py > $OUT/$T.log 2>&1
  echo "$T rc=$?" >> $OUT/$T.log
  echo "== $T"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|sanitize workload|rc=|Error|Hazard" $OUT/$T.log | head -8
done
