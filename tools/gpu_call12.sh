#!/bin/bash
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm --format=csv > $OUT/smi12.txt
timeout 400 python bench.py > $OUT/bench12_128f.json 2> $OUT/bench12_128f.err
timeout 400 python bench.py --set 192f --count 16384 --no-cpu-baseline --steps 5 > $OUT/bench12_192f.json 2> $OUT/bench12_192f.err
timeout 600 python bench.py --set 256f --count 16384 --no-cpu-baseline --steps 5 > $OUT/bench12_256f.json 2> $OUT/bench12_256f.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench12_ref.json 2> $OUT/bench12_ref.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches12.csv python tools/ncu_target.py --set 128f --count 4096 --runs 2 --mode 0 > $OUT/launches12.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tree_sign -c 1 -o /tmp/tree12 -f python tools/ncu_target.py --set 128f --count 4096 --runs 1 --mode 1 > $OUT/ncu12.log 2>&1
ncu -i /tmp/tree12.ncu-rep --page raw --csv > $OUT/tree12_raw.csv 2>&1
ncu -i /tmp/tree12.ncu-rep --page details --csv > $OUT/tree12_details.csv 2>&1
ncu -i /tmp/tree12.ncu-rep --page source --csv > $OUT/tree12_source.csv 2>&1
timeout 900 ncu --set full --clock-control none -k regex:fors_sign -c 1 -o /tmp/fors12 -f python tools/ncu_target.py --set 192f --count 4096 --runs 1 --mode 1 > $OUT/ncu12f.log 2>&1
ncu -i /tmp/fors12.ncu-rep --page raw --csv > $OUT/fors12_raw.csv 2>&1
du -sh $OUT
