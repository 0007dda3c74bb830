#!/bin/bash
# Per-launch ablations of the C1 / C2 M=1 launches in a graph (diag build)
O=gpurun_out/${1:-abl}; mkdir -p $O
(
export FLUTE_LIB=paper_2407_10960_b200/libflute_b200_diag.so
for c in "1 4096 4096 4 128" "1 4096 14336 3 128"; do
  echo "== ring GRAPH $c"; GRAPH=1 STAGES=1 timeout 120 python tools/timeline_ring.py $c 8 | head -14
  for d in 0 32 64 16 4 8 2 1 127; do
    echo -n "DIAG=$d  "; FLUTE_DIAG=$d timeout 120 python tools/graph_vs_eager.py $c
  done
  echo -n "NO_CLUSTER "; FLUTE_NO_CLUSTER=1 timeout 120 python tools/graph_vs_eager.py $c
  echo -n "NO_PDL "; FLUTE_NO_PDL=1 timeout 120 python tools/graph_vs_eager.py $c
done
) > $O/out.txt 2>&1; cat $O/out.txt
