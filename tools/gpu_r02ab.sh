#!/bin/bash
# tree_small_batch (warp-shuffle Merkle for small graphs): suite, latency table.
OUT=gpurun_out/r02ab; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest.txt 2>&1; tail -2 $OUT/pytest.txt
timeout 600 python tools/latency_probe.py > $OUT/latency.txt 2>&1; cat $OUT/latency.txt | cut -c1-110
