#!/bin/bash
# TS-kernel iteration: GPU tests under a hard timeout, then per-case timings.
TAG=${1:-ts}
O=gpurun_out/$TAG; mkdir -p $O
(
if [ -z "$NOTEST" ]; then
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 -k "${TESTS:-}" 2>&1 | tail -25
fi
for c in ${CASES:-"1 4096 4096 4 128" "16 4096 4096 4 128" "1 4096 14336 3 128" "16 4096 14336 3 128" "32 4096 14336 3 128" "1 14336 4096 3 128" "1 8192 8192 4 128" "1 8192 8192 2 128" "64 4096 4096 4 128"}; do
  timeout 100 python tools/graph_vs_eager.py $c
done
) > $O/out.txt 2>&1; cat $O/out.txt
