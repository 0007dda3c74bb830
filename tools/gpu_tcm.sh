#!/bin/bash
# tcgen05 kernel with several MMA issuer warps: parity + configs[4] + small M
O=gpurun_out/${1:-tcm}; mkdir -p $O
(
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q --timeout 60 -k "tcgen05 or tc_" 2>&1 | tail -3
timeout 200 python tools/perf_tc.py
for c in "64 4096 14336 3 128" "32 4096 14336 3 128" "16 4096 14336 3 128" "32 14336 4096 3 128" "16 4096 4096 4 128" "32 4096 4096 4 128"; do
  echo -n "mma   "; timeout 60 python tools/graph_vs_eager.py $c
  echo -n "tc32  "; FLUTE_TC_MIN_M=16 FLUTE_TC_BN=32 timeout 60 python tools/graph_vs_eager.py $c
  echo -n "tc64  "; FLUTE_TC_MIN_M=16 FLUTE_TC_BN=64 timeout 60 python tools/graph_vs_eager.py $c
done
) > $O/out.txt 2>&1; cat $O/out.txt
