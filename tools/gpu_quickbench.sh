#!/bin/bash
O=gpurun_out/${1:-qb}; mkdir -p $O
(
timeout 900 python -m pytest tests/ -m gpu -x -q --timeout 600 2>&1 | tail -2
timeout 600 python bench.py --no-cpu > $O/bench.json 2> $O/bench.err; head -c 300 $O/bench.json; echo
timeout 600 python bench.py --workload sweep --no-cpu > $O/bench_sweep.json 2> $O/bench_sweep.err; head -c 200 $O/bench_sweep.json; echo
) > $O/out.txt 2>&1; cat $O/out.txt
