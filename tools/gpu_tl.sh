#!/bin/bash
# Steady-state timelines (diag build) of chained launches + ablations in a graph.
TAG=${1:-tl}
O=gpurun_out/$TAG; mkdir -p $O
(
export FLUTE_LIB=paper_2407_10960_b200/libflute_b200_diag.so
for c in ${CASES:-"1 4096 4096 4 128" "1 4096 14336 3 128"}; do
  echo "== ring GRAPH $c"; GRAPH=1 STAGES=1 timeout 120 python tools/timeline_ring.py $c 8
  for d in 1 16 17 3 15 127; do
    echo "== FLUTE_DIAG=$d $c"; FLUTE_DIAG=$d timeout 120 python tools/graph_vs_eager.py $c
  done
done
) > $O/tl.txt 2>&1
cat $O/tl.txt
