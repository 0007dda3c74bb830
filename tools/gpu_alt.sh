#!/bin/bash
O=gpurun_out/${1:-alt}; mkdir -p $O
(
for c in "4 4096 14336 3 128" "4 14336 4096 3 128" "1 14336 4096 3 128" "8 4096 14336 3 128" "16 4096 4096 4 128" "16 4096 14336 3 128" "16 14336 4096 3 128"; do
  echo -n "base "; timeout 60 python tools/graph_vs_eager.py $c
  echo -n "alt  "; FLUTE_TRY_ALT=1 timeout 60 python tools/graph_vs_eager.py $c
done
) > $O/out.txt 2>&1; cat $O/out.txt
