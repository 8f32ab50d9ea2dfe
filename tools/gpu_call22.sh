#!/bin/bash
OUT=gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/tests22.txt 2>&1
for s in 128f 192f 256f; do for v in 0 1; do
  timeout 120 python tools/ncu_target.py --set $s --count 4096 --runs 3 --mode 1 --variant $v > $OUT/var22_${s}_$v.txt 2>&1
done; done
timeout 1500 python tools/tune_all.py --out $OUT/tuning22.json > $OUT/tune22.txt 2>&1
cp $OUT/tuning22.json paper_2512_23969_b200/b200_tuned.json
timeout 400 python bench.py > $OUT/bench22_128f.json 2> $OUT/bench22_128f.err
timeout 400 python bench.py --set 192f --count 16384 --no-cpu-baseline --steps 5 > $OUT/bench22_192f.json 2> $OUT/bench22_192f.err
timeout 600 python bench.py --set 256f --count 16384 --no-cpu-baseline --steps 5 > $OUT/bench22_256f.json 2> $OUT/bench22_256f.err
