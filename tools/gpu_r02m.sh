#!/bin/bash
# compute-sanitizer on smoke() with the round-2 kernels; ncu launch list of the bench command itself.
OUT=gpurun_out/r02m; mkdir -p $OUT
for t in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $t --error-exitcode 9 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$t.txt 2>&1; echo "$t rc=$?" >> $OUT/rc.txt
done
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_bench.csv python bench.py --single-set --steps 2 --warmup 1 --no-cpu-baseline --check 2 > $OUT/bench_under_ncu.log 2>&1
cat $OUT/rc.txt
