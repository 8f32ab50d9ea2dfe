#!/bin/bash
# verify with T_len after the chain loop (lockstep blocks) vs streamed inside the divergent branch (HEAD).
OUT=gpurun_out/r02av; mkdir -p $OUT
for r in 1 2; do
for lib in paper_2512_23969_b200/libherosign_old.so paper_2512_23969_b200/libherosign_b200.so; do
  for c in 16384 65536; do
    echo "$lib $c $(HERO_SIGN_LIB=$lib timeout 600 python tools/verify_rate.py --count $c --reps 3 | tr '\n' ' ')" >> $OUT/verify_ab.txt
  done
done
done
cat $OUT/verify_ab.txt
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest.txt 2>&1; tail -2 $OUT/pytest.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:verify_thread -c 1 -o $OUT/verify128f -f python tools/ncu_verify.py > $OUT/ncu.log 2>&1
