#!/bin/bash
# verify: chain-start prefix 1 round (rounds 0-3 per layer) vs 5 rounds per chain start (HEAD).
OUT=gpurun_out/r02bq; mkdir -p $OUT
for r in 1 2; do
for lib in paper_2512_23969_b200/libherosign_old.so paper_2512_23969_b200/libherosign_b200.so; do
  for c in 16384 65536; do
    echo "$lib $c $(HERO_SIGN_LIB=$lib timeout 600 python tools/verify_rate.py --count $c --reps 3 | tr '\n' ' ')" >> $OUT/verify_ab.txt
  done
done
done
cat $OUT/verify_ab.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "verify or corrupt" > $OUT/pytest.txt 2>&1; tail -2 $OUT/pytest.txt
