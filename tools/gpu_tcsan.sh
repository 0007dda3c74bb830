#!/bin/bash
# full GPU tests + compute-sanitizer (racecheck / synccheck / memcheck) of the tcgen05 cases
O=gpurun_out/${1:-tcsan}; mkdir -p $O
(
timeout 900 python -m pytest tests/ -m gpu -x -q --timeout 600 2>&1 | tail -3
for tool in racecheck synccheck memcheck; do
  for c in tcgen05 tcgen05_bn256 tcgen05_bn32; do
    echo "== $tool $c"
    timeout 600 compute-sanitizer --tool $tool --target-processes all --print-limit 20 \
      python tools/sanitize_cases.py $c 2>&1 | grep -v "^========= COMPUTE-SANITIZER$" | tail -4
  done
done
) > $O/out.txt 2>&1; cat $O/out.txt
