#!/bin/bash
# W3 lane-word layout: GPU tests + headline per-case graph timings + bench line
O=gpurun_out/${1:-w3}; mkdir -p $O
(
timeout 900 python -m pytest tests/ -m gpu -x -q --timeout 600 2>&1 | tail -5
for c in "1 4096 4096 4 128" "16 4096 4096 4 128" "1 4096 14336 3 128" "4 4096 14336 3 128" "16 4096 14336 3 128" "32 4096 14336 3 128" "1 14336 4096 3 128" "4 14336 4096 3 128" "16 14336 4096 3 128" "32 14336 4096 3 128"; do
  timeout 60 python tools/graph_vs_eager.py $c
done
timeout 600 python bench.py --no-cpu > $O/bench.json 2> $O/bench.err; tail -c 3000 $O/bench.json
) > $O/out.txt 2>&1; cat $O/out.txt
