#!/bin/bash
OUT=gpurun_out/r02bb; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "corrupt" > $OUT/pytest_corrupt.txt 2>&1; tail -3 $OUT/pytest_corrupt.txt
