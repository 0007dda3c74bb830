#!/bin/bash
# cluster Stream-K: parity + headline per-case timings + 70B + bench
O=gpurun_out/${1:-csk}; mkdir -p $O
(
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q --timeout 300 -k "cluster" 2>&1 | tail -3
timeout 900 python -m pytest tests/ -m gpu -x -q --timeout 600 2>&1 | tail -3
for c in "1 4096 4096 4 128" "16 4096 4096 4 128" "1 4096 14336 3 128" "4 4096 14336 3 128" "16 4096 14336 3 128" "32 4096 14336 3 128" "1 14336 4096 3 128" "32 14336 4096 3 128" "1 8192 28672 4 128" "32 4096 14336 4 128"; do
  timeout 60 python tools/graph_vs_eager.py $c
done
timeout 600 python bench.py --no-cpu > $O/bench.json 2> $O/bench.err; head -c 400 $O/bench.json
) > $O/out.txt 2>&1; cat $O/out.txt
