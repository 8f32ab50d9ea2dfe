#!/bin/bash
OUT=gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/tests20.txt 2>&1
for s in 128f 192f 256f; do for v in 0 1; do
  timeout 120 python tools/ncu_target.py --set $s --count 4096 --runs 3 --mode 1 --variant $v > $OUT/var20_${s}_$v.txt 2>&1
done; done
