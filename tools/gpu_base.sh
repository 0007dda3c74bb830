#!/bin/bash
# Baseline call of a session: per-case graph/eager timings + ncu source-level
# capture of the two C1/C2 M=1 kernels with SASS hotspots.
TAG=${1:-base}
O=gpurun_out/$TAG; mkdir -p $O
(
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
for c in "1 4096 4096 4 128" "16 4096 4096 4 128" "1 4096 14336 3 128" "4 4096 14336 3 128" "16 4096 14336 3 128" "32 4096 14336 3 128" "1 14336 4096 3 128" "32 14336 4096 3 128" "1 8192 8192 2 128" "1 8192 8192 4 128"; do
  timeout 100 python tools/graph_vs_eager.py $c
done
) > $O/out.txt 2>&1
bash tools/gpu_ncu.sh $TAG/ncu "1 4096 14336 3 128" "1 4096 4096 4 128" >> $O/out.txt 2>&1
for f in $O/ncu/prof_*.ncu-rep; do python tools/ncu_hotspots.py $f 40 >> $O/hot.txt 2>&1; python tools/ncu_summary.py $f >> $O/sum.txt 2>&1; done
cat $O/out.txt
