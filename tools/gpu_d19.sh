timeout 600 python -m pytest tests/test_gpu_parity.py -q -x --timeout 300 2>&1 | tail -2
for c in "1 4096 4096 4 128" "1 4096 14336 3 128" "16 4096 14336 3 128" "32 4096 14336 3 128" "1 14336 4096 3 128"; do timeout 60 python tools/graph_vs_eager.py $c; done 2>&1 | sed 's/R=12 workers=default pdl=on://'
export FLUTE_LIB=paper_2407_10960_b200/libflute_b200_diag.so
for d in 15 0; do echo "== DIAG=$d"; FLUTE_DIAG=$d timeout 100 python tools/timeline.py 1 4096 14336 3 128; done
