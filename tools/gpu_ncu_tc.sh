#!/bin/bash
# ncu --set full of the tcgen05 kernel at configs[4] sizes + the M<=32 kernel headline cases.
O=gpurun_out/${TAG:-ncu}; mkdir -p $O
for c in "512 8192 8192 4 128" "512 4096 4096 4 128" "128 4096 4096 4 128"; do
  t=$(echo $c | tr ' ' '_')
  NCU_PROFILING=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:qgemm_tc -s 2 -c 1 \
    -o $O/prof_tc_$t python tools/profile_case.py $c 4 > $O/ncu_tc_$t.log 2>&1
done
python tools/ncu_summary.py $O/prof_tc_*.ncu-rep > $O/ncu_tc_summary.txt 2>&1
cat $O/ncu_tc_summary.txt
