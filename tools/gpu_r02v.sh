#!/bin/bash
# Latency changes (Merkle levels in thread-local memory + leaf prefetch, T_len / T_k prefetch, unrolled out-of-line
# prep compression): GPU suite, then interleaved A/B old / compact-prep / new on small and large batches.
OUT=gpurun_out/r02v; mkdir -p $OUT
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/pytest.txt 2>&1; tail -2 $OUT/pytest.txt
timeout 1500 python tools/lat_ab.py --libs paper_2512_23969_b200/libherosign_old.so,paper_2512_23969_b200/libherosign_compact.so,paper_2512_23969_b200/libherosign_b200.so --rounds 3 > $OUT/lat_ab.txt 2>&1
cat $OUT/lat_ab.txt
