#!/bin/bash
# Concurrency test; small-batch latency breakdown (device graph vs public call) and the 1-message launch list.
OUT=gpurun_out/r02s; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_edge.py -m gpu -x -q -k concurrent > $OUT/pytest_concurrent.txt 2>&1; tail -2 $OUT/pytest_concurrent.txt
timeout 600 python tools/latency_probe.py > $OUT/latency.txt 2>&1; cat $OUT/latency.txt
for s in 128f 256f; do
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_1msg_$s.csv python tools/ncu_target.py --set $s --count 1 --runs 2 --mode 0 > $OUT/ncu_1msg_$s.log 2>&1
python tools/launch_summary.py $OUT/launches_1msg_$s.csv 2>&1 | head -40
done
