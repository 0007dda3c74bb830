#!/bin/bash
O=gpurun_out/${1:-wk4}; mkdir -p $O
(
echo "== kWK=2 (product)"; timeout 200 python tools/perf_tc.py
echo "== kWK=4"; FLUTE_LIB=paper_2407_10960_b200/libflute_b200_wk4.so timeout 200 python tools/perf_tc.py
for c in "32 4096 14336 3 128" "16 4096 14336 3 128"; do
  echo -n "tc32 wk2 "; FLUTE_TC_MIN_M=16 FLUTE_TC_BN=32 timeout 60 python tools/graph_vs_eager.py $c
  echo -n "tc32 wk4 "; FLUTE_LIB=paper_2407_10960_b200/libflute_b200_wk4.so FLUTE_TC_MIN_M=16 FLUTE_TC_BN=32 timeout 60 python tools/graph_vs_eager.py $c
done
) > $O/out.txt 2>&1; cat $O/out.txt
