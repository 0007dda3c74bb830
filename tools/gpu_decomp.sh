#!/bin/bash
O=gpurun_out/${1:-decomp}; mkdir -p $O
(
for c in "1 4096 4096 4 128" "16 4096 4096 4 128" "4 4096 14336 3 128" "16 4096 14336 3 128" "32 4096 14336 3 128" "1 14336 4096 3 128" "4 14336 4096 3 128" "16 14336 4096 3 128" "32 14336 4096 3 128"; do
  echo "### $c"
  timeout 60 python tools/graph_vs_eager.py $c | sed 's/^/default  /'
  WORKERS=296 timeout 60 python tools/graph_vs_eager.py $c | sed "s/^/sk296  /"
  for cl in 1 2 4 8; do FLUTE_FORCE_CLUSTER=$cl timeout 60 python tools/graph_vs_eager.py $c | sed "s/^/cl$cl  /"; done
done 2>&1 | sed 's/M=[0-9]* K=[0-9]* N=[0-9]* W[0-9]g128 R=12 workers=[a-z0-9]* pdl=on://'
) > $O/out.txt 2>&1; cat $O/out.txt
