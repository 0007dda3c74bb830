#!/bin/bash
# A/B of an env switch on per-case graph timings (+ optional GPU tests first).
# usage: TAG=x AB_ENV=FLUTE_NO_PRE TESTS="..." bash tools/gpu_ab.sh
O=gpurun_out/${TAG:-ab}; mkdir -p $O
(
if [ -n "$TESTS" ]; then timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 -k "$TESTS" 2>&1 | tail -8; fi
if [ -n "$ALLTESTS" ]; then timeout 1200 python -m pytest tests -m gpu -x -q --timeout 600 2>&1 | tail -8; fi
for c in ${CASES:-"1 4096 4096 4 128" "16 4096 4096 4 128" "1 4096 14336 3 128" "4 4096 14336 3 128" "16 4096 14336 3 128" "32 4096 14336 3 128" "1 14336 4096 3 128" "32 14336 4096 3 128"}; do
  timeout 100 python tools/graph_vs_eager.py $c
  [ -n "$AB_ENV" ] && env $AB_ENV=1 timeout 100 python tools/graph_vs_eager.py $c | sed "s/^/[$AB_ENV] /"
done
) > $O/out.txt 2>&1; cat $O/out.txt
