#!/bin/bash
O=gpurun_out/${1:-alt2}; mkdir -p $O
(
for c in "1 4096 4096 4 128" "1 8192 8192 4 128" "1 8192 28672 4 128" "4 8192 8192 4 128" "1 8192 8192 2 128" "4 8192 8192 2 128"; do
  echo -n "base "; timeout 60 python tools/graph_vs_eager.py $c
  echo -n "alt  "; FLUTE_TRY_ALT=1 timeout 60 python tools/graph_vs_eager.py $c
done
) > $O/out.txt 2>&1; cat $O/out.txt
