#!/bin/bash
# ncu --set full of the tcgen05 kernel (configs[4] shapes)
O=gpurun_out/${1:-ncutc}; mkdir -p $O
for c in "128 8192 8192 4 128" "512 8192 8192 4 128" "64 4096 4096 4 128"; do
  tag=$(echo $c | tr ' ' '_')
  NCU_PROFILING=1 timeout 300 ncu --set full --clock-control none -k regex:qgemm_tc -s 3 -c 1 -o $O/prof_$tag python tools/profile_case.py $c 6 > $O/ncu_$tag.log 2>&1
done
for f in $O/prof_*.ncu-rep; do python tools/ncu_summary.py $f; done > $O/sum.txt 2>&1
grep -E "==|duration|issue_active|pipe_tc_cycles_active.avg.pct_of_peak_sustained_active" $O/sum.txt
