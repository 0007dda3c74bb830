timeout 900 python -m pytest tests/ -m gpu -x -q --timeout 600 2>&1 | tail -3
for c in "1 4096 4096 4 128" "16 4096 4096 4 128" "1 4096 14336 3 128" "16 4096 14336 3 128" "32 4096 14336 3 128" "1 14336 4096 3 128"; do timeout 100 python tools/graph_vs_eager.py $c; done
export FLUTE_LIB=paper_2407_10960_b200/libflute_b200_diag.so
for d in 1 17 16; do echo "== DIAG=$d"; FLUTE_DIAG=$d timeout 100 python tools/graph_vs_eager.py 1 4096 4096 4 128; done
