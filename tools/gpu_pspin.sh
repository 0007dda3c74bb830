#!/bin/bash
O=gpurun_out/${1:-pspin}; mkdir -p $O
(
for c in "1 4096 4096 4 128" "16 4096 4096 4 128" "1 4096 14336 3 128" "4 4096 14336 3 128" "16 4096 14336 3 128" "32 4096 14336 3 128" "1 14336 4096 3 128" "32 14336 4096 3 128"; do
  echo -n "sleep "; timeout 60 python tools/graph_vs_eager.py $c
  echo -n "spin  "; FLUTE_LIB=paper_2407_10960_b200/libflute_b200_pspin.so timeout 60 python tools/graph_vs_eager.py $c
done
) > $O/out.txt 2>&1; cat $O/out.txt
