#!/bin/bash
# Bench lines (all sets, CPU baselines), reference arm, launch lists per set, full capture of tree_chain 128f.
OUT=gpurun_out/r02f; mkdir -p $OUT
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.txt 2>&1
for s in "128f 4096" "192f 16384" "256f 16384"; do set -- $s
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$1.csv python tools/ncu_target.py --set $1 --count $2 --runs 2 --mode 0 > $OUT/launches_$1.log 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tree_chain -c 1 -o $OUT/tree_chain128f -f python tools/ncu_target.py --set 128f --count 4096 --runs 1 --mode 1 > $OUT/ncu_full.log 2>&1
ls -la $OUT
