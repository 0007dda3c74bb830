#!/bin/bash
# Round checkpoint: tests, bench (both arms), launch list, ncu of the top kernels, sweep + tc workloads
TAG=${1:-r2z}
O=gpurun_out/$TAG; mkdir -p $O
bash tools/gpu_round.sh $TAG > $O/round.txt 2>&1
timeout 600 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err
timeout 900 python bench.py --workload sweep --no-cpu > $O/bench_sweep.json 2> $O/bench_sweep.err
timeout 600 python bench.py --workload tc --no-cpu > $O/bench_tc.json 2> $O/bench_tc.err
timeout 600 python bench.py --workload 70b --no-cpu > $O/bench_70b.json 2> $O/bench_70b.err
for f in $O/*.ncu-rep; do python tools/ncu_summary.py $f >> $O/ncu_summary.txt 2>&1; python tools/ncu_stallmix.py $f >> $O/ncu_stall.txt 2>&1; done
python tools/launch_share.py $O/launches.csv > $O/launch_share.txt 2>&1
tail -5 $O/round.txt; head -c 300 $O/bench.json
