#!/bin/bash
OUT=gpurun_out/r02bp; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_fuzz.py -m gpu -x -q > $OUT/pytest.txt 2>&1; tail -3 $OUT/pytest.txt
