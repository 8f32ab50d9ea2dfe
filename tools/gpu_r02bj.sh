#!/bin/bash
OUT=gpurun_out/r02bj; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "batch_size_rules" > $OUT/pytest.txt 2>&1; tail -3 $OUT/pytest.txt
