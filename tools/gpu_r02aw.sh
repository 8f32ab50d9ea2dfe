#!/bin/bash
# verify (T_len after the chain loop): native vs Mx<248> SHA path, 16384 / 65536 / 262144.
OUT=gpurun_out/r02aw; mkdir -p $OUT
for r in 1 2; do
for lib in paper_2512_23969_b200/libherosign_b200.so paper_2512_23969_b200/libherosign_vmx.so; do
  for c in 16384 65536 262144; do
    echo "$lib $c $(HERO_SIGN_LIB=$lib timeout 600 python tools/verify_rate.py --count $c --reps 3 | tr '\n' ' ')" >> $OUT/verify_ab.txt
  done
done
done
cat $OUT/verify_ab.txt
