#!/bin/bash
OUT=gpurun_out/r02b; mkdir -p $OUT
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/pytest.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.txt 2>&1
timeout 600 python bench.py --single-set --no-cpu-baseline > $OUT/bench.json 2> $OUT/bench.err
timeout 600 python bench.py --single-set --no-cpu-baseline --set 256f --count 16384 --steps 5 > $OUT/bench256.json 2> $OUT/bench256.err
tail -3 $OUT/pytest.txt
