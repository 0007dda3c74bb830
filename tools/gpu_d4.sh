for c in "1 4096 4096 4 128" "1 4096 14336 3 128" "16 4096 14336 3 128" "32 4096 14336 3 128"; do timeout 100 python tools/graph_vs_eager.py $c; done
export FLUTE_LIB=paper_2407_10960_b200/libflute_b200_diag.so
echo "== workers=1 DIAG=15"; WORKERS=1 FLUTE_DIAG=15 timeout 100 python tools/graph_vs_eager.py 1 4096 4096 4 128
for c in "1 4096 4096 4 128" "1 4096 14336 3 128"; do echo "== DIAG=15 $c"; FLUTE_DIAG=15 timeout 100 python tools/graph_vs_eager.py $c; done
