#!/bin/bash
O=gpurun_out/${1:-wsweep2}; mkdir -p $O
(
for c in "1 14336 4096 3 128" "4 14336 4096 3 128" "16 14336 4096 3 128" "1 4096 4096 4 128" "16 4096 4096 4 128"; do
  echo "### $c"
  timeout 60 python tools/graph_vs_eager.py $c | sed 's/^/default /'
  for w in 256 288 296; do WORKERS=$w timeout 60 python tools/graph_vs_eager.py $c | sed "s/^/w$w /"; done
done 2>&1 | sed 's/M=[0-9]* K=[0-9]* N=[0-9]* W[0-9]g[0-9]* R=12 workers=[a-z0-9]* pdl=on://; s/eager [0-9.]* us ([0-9]* GB\/s)  //'
) > $O/out.txt 2>&1; cat $O/out.txt
