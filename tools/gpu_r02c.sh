#!/bin/bash
# Round-2 first GPU pass: GPU suite, smoke, default bench line (all sets + CPU baselines), launch list.
OUT=gpurun_out/r02c; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/smi.txt
timeout 1500 python -m pytest tests -m gpu -x -q --durations=25 > $OUT/pytest.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.txt 2>&1
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_128f.csv python tools/ncu_target.py --set 128f --count 4096 --runs 2 --mode 0 > $OUT/launches.log 2>&1
tail -5 $OUT/pytest.txt
