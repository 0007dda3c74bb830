#!/bin/bash
# A/B two builds of the library on the same box: GPU parity of the current
# build, then graph timings of each case with BASE (libflute_b200_base.so) and NEW.
O=gpurun_out/${1:-ab}; mkdir -p $O
(
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 2>&1 | tail -2
CASES=${CASES:-"1 4096 14336 3 128|1 14336 4096 3 128|4 4096 14336 3 128|16 4096 14336 3 128|16 14336 4096 3 128|32 4096 14336 3 128|32 14336 4096 3 128|1 4096 4096 4 128"}
IFS='|'; for c in $CASES; do
  IFS=' '
  for rep in 1 2; do
    echo "BASE $(FLUTE_LIB=paper_2407_10960_b200/libflute_b200_base.so timeout 60 python tools/graph_vs_eager.py $c)"
    echo "NEW  $(timeout 60 python tools/graph_vs_eager.py $c)"
  done
  IFS='|'
done
) > $O/out.txt 2>&1; cat $O/out.txt
