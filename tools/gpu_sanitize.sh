#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over every device
# protocol (tools/sanitize_cases.py), one process per case.
O=gpurun_out/${TAG:-san}; mkdir -p $O
for tool in memcheck racecheck synccheck; do
  for c in streamk streamk_w3 ticket cluster tcgen05 tcgen05_bn256 tcgen05_bn32 default default_m32; do
    echo "== $tool $c"
    timeout 600 compute-sanitizer --tool $tool --target-processes all --print-limit 20 \
      python tools/sanitize_cases.py $c 2>&1 | grep -v "^========= COMPUTE-SANITIZER$" | tail -6
  done
done > $O/sanitizer.txt 2>&1
cat $O/sanitizer.txt
