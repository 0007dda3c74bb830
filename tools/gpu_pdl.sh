#!/bin/bash
# PDL in eager launches vs captured graphs
for c in "1 4096 14336 3 128" "1 4096 4096 4 128"; do
  for rep in 1 2; do
    echo "PDL   $(timeout 60 python tools/graph_vs_eager.py $c)"
    echo "NOPDL $(FLUTE_NO_PDL=1 timeout 60 python tools/graph_vs_eager.py $c)"
  done
done
