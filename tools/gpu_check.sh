#!/bin/bash
# One gpurun call: GPU parity tests (hard timeout), then per-case graph timings.
# usage (here): gpurun --timeout 1800 -- 'bash tools/gpu_check.sh TAG'
TAG=${1:-chk}
O=gpurun_out/$TAG; mkdir -p $O
(
if [ -z "$NOTEST" ]; then
timeout 1200 python -m pytest tests -m gpu -x -q --timeout 600 -k "${TESTS:-}" 2>&1 | tail -15
fi
for c in ${CASES:-"1 4096 4096 4 128" "16 4096 4096 4 128" "1 4096 14336 3 128" "16 4096 14336 3 128" "32 4096 14336 3 128" "1 14336 4096 3 128" "1 8192 8192 4 128" "1 8192 8192 2 128" "1 8192 28672 4 128"}; do
  timeout 100 python tools/graph_vs_eager.py $c
done
) > $O/out.txt 2>&1; cat $O/out.txt
