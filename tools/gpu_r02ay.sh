#!/bin/bash
# Final pass after the verify restructure: suite, smoke, config-5 stress (verify rates), compute-sanitizer on smoke.
OUT=gpurun_out/r02ay; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest.txt 2>&1; tail -2 $OUT/pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.txt 2>&1; tail -1 $OUT/smoke.txt
timeout 2400 python tools/stress_c5.py > $OUT/stress_c5.txt 2>&1; grep '"set"' $OUT/stress_c5.txt
for t in memcheck racecheck; do
  timeout 900 compute-sanitizer --tool $t --error-exitcode 9 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$t.txt 2>&1; echo "smoke $t rc=$?"
done
