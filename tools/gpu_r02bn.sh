#!/bin/bash
# public call without the redundant end-of-call stream syncs: latency table, GPU suite.
OUT=gpurun_out/r02bn; mkdir -p $OUT
timeout 600 python tools/latency_probe.py --counts 1,4,64 > $OUT/latency.txt 2>&1; cut -c1-160 $OUT/latency.txt
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest.txt 2>&1; tail -2 $OUT/pytest.txt
