OUT=gpurun_out/${OUT:-r02c}; mkdir -p $OUT
timeout 300 python tools/k1_bench.py > $OUT/k1_bench_team.jsonl 2>&1
CRT_K1_TEAM=0 timeout 300 python tools/k1_bench.py > $OUT/k1_bench_rolled.jsonl 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/k1_ncu_launches.csv python tools/k1_time.py > /dev/null 2>&1
cat $OUT/k1_bench_team.jsonl $OUT/k1_bench_rolled.jsonl
grep -E "k1_team|k1_rolled" $OUT/k1_ncu_launches.csv | awk -F'","' '{print $5, $NF}' | sort | uniq -c | head -30
