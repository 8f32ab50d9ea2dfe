#!/bin/bash
OUT=gpurun_out/r02aj; mkdir -p $OUT
timeout 600 python tools/latency_probe.py --counts 1,4,64,4096 > $OUT/latency.txt 2>&1; cut -c1-175 $OUT/latency.txt
