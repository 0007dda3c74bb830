#!/bin/bash
# cluster Stream-K regression hunt: HEAD lib vs current, forced decompositions, timelines
O=gpurun_out/${1:-csk2}; mkdir -p $O
(
for c in "1 4096 4096 4 128" "1 4096 14336 3 128"; do
  echo "== $c"
  echo -n "head default  "; FLUTE_LIB=paper_2407_10960_b200/libflute_b200_head.so timeout 60 python tools/graph_vs_eager.py $c
  echo -n "cur default   "; timeout 60 python tools/graph_vs_eager.py $c
  echo -n "head C4       "; FLUTE_FORCE_CLUSTER=4 FLUTE_LIB=paper_2407_10960_b200/libflute_b200_head.so timeout 60 python tools/graph_vs_eager.py $c
  echo -n "cur C4 T1     "; FLUTE_FORCE_CLUSTER=4 timeout 60 python tools/graph_vs_eager.py $c
  echo -n "cur C1 T1     "; FLUTE_FORCE_CLUSTER=1 timeout 60 python tools/graph_vs_eager.py $c
  echo -n "cur C5 T4     "; FLUTE_FORCE_CLUSTER=5 FLUTE_FORCE_CTILES=4 timeout 60 python tools/graph_vs_eager.py $c
  echo -n "cur C2 T1     "; FLUTE_FORCE_CLUSTER=2 timeout 60 python tools/graph_vs_eager.py $c
done
FLUTE_LIB=paper_2407_10960_b200/libflute_b200_diag.so FLUTE_FORCE_CLUSTER=5 FLUTE_FORCE_CTILES=4 GRAPH=1 timeout 120 python tools/timeline_ring.py 1 4096 14336 3 128 8 2>/dev/null | sed -n '1,30p'
FLUTE_LIB=paper_2407_10960_b200/libflute_b200_diag.so GRAPH=1 timeout 120 python tools/timeline_ring.py 1 4096 4096 4 128 8 2>/dev/null | sed -n '1,30p'
) > $O/out.txt 2>&1; cat $O/out.txt
