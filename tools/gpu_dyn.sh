#!/bin/bash
# dynamic item mode + W3 lane words: parity (GPU tests) + per-case timings vs the static decomposition
O=gpurun_out/${1:-dyn}; mkdir -p $O
(
timeout 900 python -m pytest tests/ -m gpu -x -q --timeout 600 2>&1 | tail -15
for c in "1 4096 4096 4 128" "1 4096 14336 3 128" "4 4096 14336 3 128" "16 4096 14336 3 128" "32 4096 14336 3 128" "1 14336 4096 3 128" "32 14336 4096 3 128" "1 8192 8192 4 128" "8 4096 14336 3 128" "1 8192 28672 4 128"; do
  echo "== $c"
  FLUTE_NO_DYN=1 timeout 60 python tools/graph_vs_eager.py $c
  timeout 60 python tools/graph_vs_eager.py $c
  FLUTE_DYN_PER=2 timeout 60 python tools/graph_vs_eager.py $c
  FLUTE_DYN_PER=8 timeout 60 python tools/graph_vs_eager.py $c
done
) > $O/out.txt 2>&1; cat $O/out.txt
