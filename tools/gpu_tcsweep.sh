#!/bin/bash
# tcgen05 decomposition sweep (BN, splits) for configs[4]
O=gpurun_out/${1:-tcsweep}; mkdir -p $O
(
for c in "64 4096 4096 4 128" "128 4096 4096 4 128" "256 4096 4096 4 128" "512 4096 4096 4 128" "128 8192 8192 4 128" "256 8192 8192 4 128"; do
  echo "### $c"
  timeout 60 python tools/graph_vs_eager.py $c | sed 's/^/default /'
  for bn in 64 128 256; do for sp in 1 2 4 6; do
    FLUTE_TC_BN=$bn FLUTE_TC_SPLITS=$sp timeout 60 python tools/graph_vs_eager.py $c | sed "s/^/bn$bn sp$sp /"
  done; done
done 2>&1 | sed 's/M=[0-9]* K=[0-9]* N=[0-9]* W[0-9]g[0-9]* R=12 workers=[a-z0-9]* pdl=on://; s/eager [0-9.]* us ([0-9]* GB\/s)  //'
) > $O/out.txt 2>&1; cat $O/out.txt
