#!/bin/bash
O=gpurun_out/${1:-tcspin}; mkdir -p $O
(
echo "== sleep (product)"; timeout 300 python tools/perf_tc.py
echo "== spin"; FLUTE_LIB=paper_2407_10960_b200/libflute_b200_tcspin.so timeout 300 python tools/perf_tc.py
for c in "32 4096 14336 3 128" "16 4096 14336 3 128"; do
  echo -n "mma   "; timeout 60 python tools/graph_vs_eager.py $c
  echo -n "tc    "; FLUTE_TC_MIN_M=16 FLUTE_TC_BN=32 timeout 60 python tools/graph_vs_eager.py $c
  echo -n "tcspin"; FLUTE_LIB=paper_2407_10960_b200/libflute_b200_tcspin.so FLUTE_TC_MIN_M=16 FLUTE_TC_BN=32 timeout 60 python tools/graph_vs_eager.py $c
done
) > $O/out.txt 2>&1; cat $O/out.txt
