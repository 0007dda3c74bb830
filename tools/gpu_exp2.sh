#!/bin/bash
# W2 replicated table + tcgen05 at M = 16 / 32 (FLUTE_TC_MIN_M, BN 32 / 64)
O=gpurun_out/${1:-exp2}; mkdir -p $O
(
timeout 900 python -m pytest tests/ -m gpu -x -q --timeout 600 2>&1 | tail -3
for c in "1 8192 8192 2 128" "16 8192 8192 2 128" "32 8192 8192 2 128" "1 8192 8192 3 128"; do timeout 60 python tools/graph_vs_eager.py $c; done
for c in "16 4096 14336 3 128" "32 4096 14336 3 128" "16 14336 4096 3 128" "32 14336 4096 3 128" "16 4096 4096 4 128" "32 4096 4096 4 128"; do
  echo "== $c"
  timeout 60 python tools/graph_vs_eager.py $c
  FLUTE_TC_MIN_M=16 FLUTE_TC_BN=32 timeout 60 python tools/graph_vs_eager.py $c
  FLUTE_TC_MIN_M=16 FLUTE_TC_BN=64 timeout 60 python tools/graph_vs_eager.py $c
  FLUTE_TC_MIN_M=16 FLUTE_TC_BN=32 FLUTE_TC_SPLITS=2 timeout 60 python tools/graph_vs_eager.py $c
done
) > $O/out.txt 2>&1; cat $O/out.txt
