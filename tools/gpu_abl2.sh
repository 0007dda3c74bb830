#!/bin/bash
# Stream-K over every slot (P = 296) vs the default, with CTA placement
O=gpurun_out/${1:-abl2}; mkdir -p $O
(
for c in "1 4096 4096 4 128" "1 4096 14336 3 128" "1 14336 4096 3 128" "4 4096 14336 3 128"; do
  echo "== $c"
  timeout 60 python tools/graph_vs_eager.py $c
  WORKERS=296 timeout 60 python tools/graph_vs_eager.py $c
  WORKERS=148 timeout 60 python tools/graph_vs_eager.py $c
  FLUTE_LIB=paper_2407_10960_b200/libflute_b200_diag.so WORKERS=296 GRAPH=1 timeout 120 python tools/timeline_ring.py $c 8 2>/dev/null | sed -n '1,14p'
done
) > $O/out.txt 2>&1; cat $O/out.txt
