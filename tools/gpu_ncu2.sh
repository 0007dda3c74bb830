#!/bin/bash
# ncu --set full of the M=16 / M=32 configs[1] launches + stall mix
TAG=${1:-ncu2}
bash tools/gpu_ncu.sh $TAG "32 4096 14336 3 128" "16 4096 14336 3 128" "1 4096 14336 3 128"
O=gpurun_out/$TAG
for f in $O/prof_*.ncu-rep; do python tools/ncu_summary.py $f >> $O/sum.txt 2>&1; python tools/ncu_stallmix.py $f >> $O/stall.txt 2>&1; python tools/ncu_hotspots.py $f 30 >> $O/hot.txt 2>&1; done
cat $O/sum.txt | grep -v "  0 \|0 %\|0 inst"
