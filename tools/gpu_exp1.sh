#!/bin/bash
# CW=8 / 148-worker launch-structure experiment (M=1 decode shapes).
O=gpurun_out/exp1; mkdir -p $O
(
for c in "1 4096 4096 4 128" "1 4096 14336 3 128" "1 14336 4096 3 128" "1 8192 8192 4 128" "1 8192 8192 2 128" "8 4096 14336 3 128"; do
  echo "== $c"
  timeout 60 python tools/graph_vs_eager.py $c
  WORKERS=148 timeout 60 python tools/graph_vs_eager.py $c
  FLUTE_M8_CW8=1 timeout 60 python tools/graph_vs_eager.py $c
  FLUTE_M8_CW8=1 WORKERS=148 timeout 60 python tools/graph_vs_eager.py $c
  FLUTE_M8_CW8=1 WORKERS=296 timeout 60 python tools/graph_vs_eager.py $c
  FLUTE_M8_CW8=4 WORKERS=148 timeout 60 python tools/graph_vs_eager.py $c
done
) > $O/out.txt 2>&1; cat $O/out.txt
