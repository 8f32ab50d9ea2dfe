#!/bin/bash
OUT=gpurun_out/r02bk; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_edge.py -m gpu -x -q -k "small_tail" > $OUT/pytest.txt 2>&1; tail -3 $OUT/pytest.txt
