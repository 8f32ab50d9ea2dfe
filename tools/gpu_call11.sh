#!/bin/bash
OUT=gpurun_out
mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/tests11.txt 2>&1
for s in 128f 192f 256f; do for v in 0 1; do
  timeout 120 python tools/ncu_target.py --set $s --count 4096 --runs 3 --mode 1 --variant $v > $OUT/var11_${s}_$v.txt 2>&1
done; done
timeout 900 python tools/tune_all.py --out $OUT/tuning11.json > $OUT/tune11.txt 2>&1
