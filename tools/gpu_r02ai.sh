#!/bin/bash
# compute-sanitizer on smoke() and on small / batch-size-rule batches with the round-2 latency kernels.
OUT=gpurun_out/r02ai; mkdir -p $OUT
for t in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $t --error-exitcode 9 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$t.txt 2>&1; echo "smoke $t rc=$?" >> $OUT/rc.txt
done
timeout 1200 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "batch_size_rules" > $OUT/rules_memcheck.txt 2>&1; echo "rules memcheck rc=$?" >> $OUT/rc.txt
cat $OUT/rc.txt; tail -3 $OUT/rules_memcheck.txt
