#!/bin/bash
# K1 team-shape sweep (dev aid): default plan vs forced W,C, single-pass teams.
for MK in "4608 3072" "4608 12288"; do
  echo "== $MK default"; timeout 60 python tools/k1_one.py $MK
  for P in "1,6" "2,4" "3,2" "4,6" "6,4" "3,8" "6,2"; do
    echo "-- plan $P fast-teams"; CRT_K1_PLAN=$P CRT_K1_FAST_TEAMS=1 timeout 60 python tools/k1_one.py $MK check 2>&1 | tail -1
  done
done
