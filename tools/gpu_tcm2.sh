#!/bin/bash
O=gpurun_out/${1:-tcm2}; mkdir -p $O
(
timeout 900 python -m pytest tests/ -m gpu -x -q --timeout 600 2>&1 | tail -3
timeout 600 python bench.py --workload tc --no-cpu > $O/bench_tc.json 2> $O/bench_tc.err; head -c 600 $O/bench_tc.json; echo
FLUTE_LIB=paper_2407_10960_b200/libflute_b200_diag.so timeout 120 python tools/tc_trace.py 128 4096 4096 4 128 2>&1 | head -24
FLUTE_LIB=paper_2407_10960_b200/libflute_b200_diag.so FLUTE_TC_MIN_M=16 FLUTE_TC_BN=32 timeout 120 python tools/tc_trace.py 32 4096 14336 3 128 2>&1 | head -24
NCU_PROFILING=1 timeout 300 ncu --set full --clock-control none -k regex:qgemm_tc -s 3 -c 1 -o $O/prof_tc_512 python tools/profile_case.py 512 8192 8192 4 128 6 > $O/ncu.log 2>&1
NCU_PROFILING=1 timeout 300 ncu --set full --clock-control none -k regex:qgemm_tc -s 3 -c 1 -o $O/prof_tc_128 python tools/profile_case.py 128 8192 8192 4 128 6 >> $O/ncu.log 2>&1
for f in $O/prof_tc_*.ncu-rep; do python tools/ncu_summary.py $f; done
) > $O/out.txt 2>&1; cat $O/out.txt
