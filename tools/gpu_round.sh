#!/bin/bash
# One gpurun call: tests, bench lines for each set, ncu launch list and a full capture of TREE_Sign.
set -x
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/smi.txt
timeout 300 python bench.py > $OUT/bench_128f.json 2> $OUT/bench_128f.err
timeout 300 python bench.py --set 192f --count 16384 --no-cpu-baseline --steps 5 > $OUT/bench_192f.json 2> $OUT/bench_192f.err
timeout 300 python bench.py --set 256f --count 8192 --no-cpu-baseline --steps 5 > $OUT/bench_256f.json 2> $OUT/bench_256f.err
for v in 0 1; do timeout 120 python tools/ncu_target.py --set 128f --count 4096 --runs 2 --mode 1 --variant $v > $OUT/variant_$v.txt 2>&1; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv python tools/ncu_target.py --set 128f --count 4096 --runs 2 --mode 0 > $OUT/launches.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tree_sign -c 1 -o $OUT/tree128f -f python tools/ncu_target.py --set 128f --count 4096 --runs 1 --mode 1 > $OUT/ncu_full.log 2>&1
ls -la $OUT
