#!/bin/bash
O=gpurun_out/${1:-alt3}; mkdir -p $O
(
for c in "32 14336 4096 3 128" "24 14336 4096 3 128" "32 8192 8192 3 128" "32 8192 8192 2 128" "32 4096 14336 3 128"; do
  echo -n "base "; timeout 60 python tools/graph_vs_eager.py $c
  echo -n "alt  "; FLUTE_TRY_ALT=1 timeout 60 python tools/graph_vs_eager.py $c
done
) > $O/out.txt 2>&1; cat $O/out.txt
