#!/bin/bash
# Diagnostics call: streaming ceiling, per-CTA timeline, graph vs eager, and
# the FLUTE_DIAG ablations (diag build).  usage: bash tools/gpu_diag.sh TAG
TAG=${1:-diag}
O=gpurun_out/$TAG
mkdir -p $O
(
echo "== tma_stream_bench"; timeout 120 tools/_build/tma_stream_bench
for c in "1 4096 4096 4 128" "1 4096 14336 3 128" "32 4096 14336 3 128"; do
  echo "== graph_vs_eager $c"; timeout 120 python tools/graph_vs_eager.py $c
done
export FLUTE_LIB=paper_2407_10960_b200/libflute_b200_diag.so
for d in 1 2 4 8 3 15; do
  for c in "1 4096 4096 4 128" "1 4096 14336 3 128"; do
    echo "== FLUTE_DIAG=$d $c"; FLUTE_DIAG=$d timeout 120 python tools/graph_vs_eager.py $c
  done
done
for c in "1 4096 4096 4 128" "1 4096 14336 3 128"; do
  echo "== timeline $c"; timeout 120 python tools/timeline.py $c --stages
done
) > $O/diag.txt 2>&1
tail -c 3000 $O/diag.txt
