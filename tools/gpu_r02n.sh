#!/bin/bash
# tree_split 1 (warp-shuffle Merkle in the leaf grid) vs 2 (leaf grid + one thread per subtree), GPU suite.
OUT=gpurun_out/r02n; mkdir -p $OUT
for s in "128f 4096" "192f 16384" "256f 16384"; do set -- $s
  timeout 600 python tools/ab_config.py --set $1 --count $2 --rounds 4 --serial --a '{"tree_split": 1}' --b '{"tree_split": 2}' >> $OUT/ab_tree_split.txt 2>&1
done
cat $OUT/ab_tree_split.txt
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/pytest.txt 2>&1; tail -3 $OUT/pytest.txt
