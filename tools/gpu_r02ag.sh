#!/bin/bash
# public-call overhead: waits / syncs only on the copy-out streams a call used; raw C call vs Python wrapper.
OUT=gpurun_out/r02ag; mkdir -p $OUT
timeout 600 python tools/latency_probe.py --counts 1,4,64 > $OUT/latency.txt 2>&1; cut -c1-150 $OUT/latency.txt
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest.txt 2>&1; tail -2 $OUT/pytest.txt
