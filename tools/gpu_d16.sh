export FLUTE_LIB=paper_2407_10960_b200/libflute_b200_diag.so
for d in 0 14 15 1; do for c in "1 4096 14336 3 128" "1 4096 4096 4 128" "32 4096 14336 3 128"; do echo "DIAG=$d $(FLUTE_DIAG=$d timeout 60 python tools/graph_vs_eager.py $c)"; done; done 2>&1 | sed 's/R=12 workers=default pdl=on://'
