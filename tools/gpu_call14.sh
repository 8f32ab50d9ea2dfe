#!/bin/bash
OUT=gpurun_out
mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/tests14.txt 2>&1
timeout 2400 python tools/stress_c5.py --messages 1048576 > $OUT/stress14.txt 2>&1
