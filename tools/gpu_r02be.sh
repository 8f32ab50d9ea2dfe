#!/bin/bash
# 1-message launch list on the final code (graph mode; serialised by ncu).
OUT=gpurun_out/r02be; mkdir -p $OUT
for s in 128f 192f 256f; do
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_1msg_$s.csv python tools/ncu_target.py --set $s --count 1 --runs 2 --mode 0 > $OUT/ncu_$s.log 2>&1
python tools/launch_summary.py $OUT/launches_1msg_$s.csv 2>&1 | head -16
done
