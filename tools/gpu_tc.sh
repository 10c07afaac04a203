OUT=gpurun_out/${OUT:-r02u}; mkdir -p $OUT
timeout 300 python tools/k1_bench.py 4608 3072 16 5 4608 12288 16 5 4608 15360 16 5 4096 3072 16 5 4608 3072 4 5 4608 3072 16 4 4608 12288 16 4 > $OUT/k1_tc.jsonl 2>&1
CRT_K1_TC=0 timeout 300 python tools/k1_bench.py 4608 3072 16 5 4608 12288 16 5 4608 15360 16 5 > $OUT/k1_team.jsonl 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
cat $OUT/k1_tc.jsonl; echo ---; cat $OUT/k1_team.jsonl; tail -25 $OUT/pytest.log
