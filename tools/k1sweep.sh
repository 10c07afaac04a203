for w in 1 2 3 4 6 8; do echo "W=$w"; CRT_K1_ROLLED=1 CRT_K1_W=$w timeout 120 python tools/quick_timing.py k1 2>&1 | grep "N0=16"; done
