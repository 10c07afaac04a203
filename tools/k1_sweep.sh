#!/bin/bash
# K1 team-shape sweep (dev aid): default plan vs forced CRT_K1_PLAN="W,C",
# rolled kernel (default) and single-pass (CRT_K1_FAST=1, W = 1 only).
for MK in "4608 3072" "4608 12288"; do
  echo "== $MK default"; timeout 60 python tools/k1_one.py $MK
  echo "-- single-pass"; CRT_K1_FAST=1 timeout 60 python tools/k1_one.py $MK check 2>&1 | tail -1
  for P in "1,6" "2,4" "3,2" "4,6" "6,4" "3,8" "8,4"; do
    echo "-- plan $P"; CRT_K1_PLAN=$P timeout 60 python tools/k1_one.py $MK check 2>&1 | tail -1
  done
done
