#!/bin/bash
# Python wrapper overhead trimmed (cached derive, int pointers): latency table, suite.
OUT=gpurun_out/r02ah; mkdir -p $OUT
timeout 600 python tools/latency_probe.py --counts 1,4,64 > $OUT/latency.txt 2>&1; cut -c1-150 $OUT/latency.txt
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest.txt 2>&1; tail -2 $OUT/pytest.txt
