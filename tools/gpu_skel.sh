#!/bin/bash
# Bisect the per-launch skeleton with FLUTE_DIAG bits (diag build), graph timings
O=gpurun_out/${1:-skel}; mkdir -p $O
(
export FLUTE_LIB=paper_2407_10960_b200/libflute_b200_diag.so
for c in "1 4096 4096 4 128" "1 4096 14336 3 128"; do
  echo "== $c"
  for d in 0 127 255 383 895 1919 2047 1663 1151; do
    echo -n "DIAG=$d  "; FLUTE_DIAG=$d timeout 60 python tools/graph_vs_eager.py $c
  done
done
) > $O/out.txt 2>&1; cat $O/out.txt
