#!/bin/bash
OUT=gpurun_out
mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/tests13.txt 2>&1
timeout 1200 python tools/tune_all.py --out $OUT/tuning13.json > $OUT/tune13.txt 2>&1
cp $OUT/tuning13.json paper_2512_23969_b200/b200_tuned.json
timeout 400 python bench.py --no-cpu-baseline > $OUT/bench13_128f.json 2> $OUT/bench13_128f.err
timeout 400 python bench.py --set 192f --count 16384 --no-cpu-baseline --steps 5 > $OUT/bench13_192f.json 2> $OUT/bench13_192f.err
timeout 600 python bench.py --set 256f --count 16384 --no-cpu-baseline --steps 5 > $OUT/bench13_256f.json 2> $OUT/bench13_256f.err
timeout 900 ncu --set full --clock-control none -k regex:fors_sign -c 1 -o /tmp/fors13 -f python tools/ncu_target.py --set 192f --count 4096 --runs 1 --mode 1 > $OUT/ncu13f.log 2>&1
ncu -i /tmp/fors13.ncu-rep --page raw --csv > $OUT/fors13_raw.csv 2>&1
