#!/bin/bash
OUT=gpurun_out
mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/tests17.txt 2>&1
timeout 400 python bench.py > $OUT/bench17_128f.json 2> $OUT/bench17_128f.err
timeout 400 python bench.py --set 192f --count 16384 --no-cpu-baseline --steps 5 > $OUT/bench17_192f.json 2> $OUT/bench17_192f.err
timeout 600 python bench.py --set 256f --count 16384 --no-cpu-baseline --steps 5 > $OUT/bench17_256f.json 2> $OUT/bench17_256f.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches17.csv python tools/ncu_target.py --set 128f --count 4096 --runs 2 --mode 0 > $OUT/launches17.log 2>&1
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke17.txt 2>&1
