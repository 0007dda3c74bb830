#!/bin/bash
# ncu --set full of one case per argument "M K N BITS GROUP" (first kernel after warm-up).
TAG=$1; shift
O=gpurun_out/$TAG; mkdir -p $O
i=0
for c in "$@"; do
  i=$((i+1))
  NCU_PROFILING=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:qgemm -s 6 -c 1 \
    -o $O/prof_$i python tools/profile_case.py $c 8 > $O/ncu_$i.log 2>&1
  echo "$c -> prof_$i: $(tail -1 $O/ncu_$i.log)"
done
