#!/bin/bash
# batched Stream-K finisher polling; epilogue sleep A/B; P = 296 vs default
O=gpurun_out/${1:-abl3}; mkdir -p $O
(
timeout 900 python -m pytest tests/ -m gpu -x -q --timeout 600 2>&1 | tail -3
for c in "1 4096 4096 4 128" "16 4096 4096 4 128" "1 4096 14336 3 128" "1 14336 4096 3 128" "4 4096 14336 3 128" "16 4096 14336 3 128" "16 14336 4096 3 128" "32 4096 14336 3 128" "32 14336 4096 3 128"; do
  echo "== $c"
  timeout 60 python tools/graph_vs_eager.py $c
  WORKERS=296 timeout 60 python tools/graph_vs_eager.py $c
  FLUTE_LIB=paper_2407_10960_b200/libflute_b200_nosleep.so timeout 60 python tools/graph_vs_eager.py $c
  FLUTE_LIB=paper_2407_10960_b200/libflute_b200_nosleep.so WORKERS=296 timeout 60 python tools/graph_vs_eager.py $c
done
FLUTE_LIB=paper_2407_10960_b200/libflute_b200_diag.so WORKERS=296 GRAPH=1 timeout 120 python tools/timeline_ring.py 1 14336 4096 3 128 8 2>/dev/null | sed -n '1,14p'
) > $O/out.txt 2>&1; cat $O/out.txt
