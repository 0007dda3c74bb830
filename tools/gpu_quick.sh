#!/bin/bash
# Quick iteration call: GPU parity tests + per-case graph/eager timings (+ timeline).
TAG=${1:-q}
O=gpurun_out/$TAG; mkdir -p $O
(
timeout 900 python -m pytest tests/ -m gpu -x -q --timeout 600 2>&1 | tail -5
for c in "1 4096 4096 4 128" "16 4096 4096 4 128" "1 4096 14336 3 128" "4 4096 14336 3 128" "16 4096 14336 3 128" "32 4096 14336 3 128" "1 14336 4096 3 128" "32 14336 4096 3 128" "1 8192 8192 2 128"; do
  timeout 100 python tools/graph_vs_eager.py $c
done
if [ -n "$TIMELINE" ]; then
  for c in "1 4096 4096 4 128" "1 4096 14336 3 128"; do
    echo "== timeline $c"; FLUTE_LIB=paper_2407_10960_b200/libflute_b200_diag.so timeout 120 python tools/timeline.py $c --stages
  done
fi
) > $O/out.txt 2>&1; cat $O/out.txt
