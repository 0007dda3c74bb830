#!/bin/bash
O=gpurun_out/${1:-sweepdec}; mkdir -p $O
(
for c in "1 8192 8192 4 128" "1 8192 8192 3 128" "1 8192 8192 2 128" "4 8192 8192 3 32" "16 8192 8192 3 128" "1 8192 28672 4 128"; do
  echo "### $c"
  timeout 60 python tools/graph_vs_eager.py $c | sed 's/^/default  /'
  WORKERS=296 timeout 60 python tools/graph_vs_eager.py $c | sed "s/^/sk296  /"
  FLUTE_FORCE_CLUSTER=4 timeout 60 python tools/graph_vs_eager.py $c | sed "s/^/cl4  /"
done 2>&1 | sed 's/M=[0-9]* K=[0-9]* N=[0-9]* W[0-9]g[0-9]* R=12 workers=[a-z0-9]* pdl=on://; s/eager [0-9.]* us ([0-9]* GB\/s)  //'
) > $O/out.txt 2>&1; cat $O/out.txt
