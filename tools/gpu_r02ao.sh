#!/bin/bash
# 128f config-5 e2e/device A/B: session-start library (648d173, its tuned config) vs current.
OUT=gpurun_out/r02ao; mkdir -p $OUT
for r in 1 2; do
  HERO_SIGN_LIB=paper_2512_23969_b200/libherosign_old.so HERO_SIGN_CONFIG=paper_2512_23969_b200/old_tuned.json timeout 900 python tools/stress_c5.py --sets 128f --messages 262144 > $OUT/old_$r.txt 2>&1; tail -1 $OUT/old_$r.txt
  timeout 900 python tools/stress_c5.py --sets 128f --messages 262144 > $OUT/new_$r.txt 2>&1; tail -1 $OUT/new_$r.txt
done
