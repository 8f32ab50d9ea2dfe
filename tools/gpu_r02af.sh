#!/bin/bash
# verify keeps the compact prologue compression: verify A/B vs HEAD, suite, latency.
OUT=gpurun_out/r02af; mkdir -p $OUT
for r in 1 2; do
for lib in paper_2512_23969_b200/libherosign_old.so paper_2512_23969_b200/libherosign_b200.so; do
  echo "$lib $(HERO_SIGN_LIB=$lib timeout 600 python tools/verify_rate.py --count 65536 --reps 3 | tr '\n' ' ')" >> $OUT/verify_ab.txt
done
done
cat $OUT/verify_ab.txt
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest.txt 2>&1; tail -2 $OUT/pytest.txt
timeout 600 python tools/latency_probe.py --counts 1,4,16 > $OUT/latency.txt 2>&1; cut -c1-110 $OUT/latency.txt
