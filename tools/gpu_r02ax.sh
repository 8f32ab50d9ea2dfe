#!/bin/bash
# verify block size 128 (current) vs 64 vs 32: SM balance of the thread-per-signature grid.
OUT=gpurun_out/r02ax; mkdir -p $OUT
for r in 1 2; do
for lib in paper_2512_23969_b200/libherosign_b200.so paper_2512_23969_b200/libherosign_vt64.so paper_2512_23969_b200/libherosign_vt32.so; do
  for c in 16384 65536; do
    echo "$lib $c $(HERO_SIGN_LIB=$lib timeout 600 python tools/verify_rate.py --count $c --reps 3 | tr '\n' ' ')" >> $OUT/verify_ab.txt
  done
done
done
cat $OUT/verify_ab.txt
