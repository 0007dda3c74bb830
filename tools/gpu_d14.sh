export FLUTE_LIB=paper_2407_10960_b200/libflute_b200_diag.so
echo "== DIAG=13 timeline"; FLUTE_DIAG=13 timeout 100 python tools/timeline.py 1 4096 14336 3 128 --stages
echo "== DIAG=0 timeline"; timeout 100 python tools/timeline.py 1 4096 14336 3 128 --stages
