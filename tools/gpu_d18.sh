export FLUTE_LIB=paper_2407_10960_b200/libflute_b200_diag.so
for d in 15 0; do echo "== DIAG=$d"; FLUTE_DIAG=$d timeout 100 python tools/timeline.py 1 4096 14336 3 128; done
echo "== DIAG=15 C1"; FLUTE_DIAG=15 timeout 100 python tools/timeline.py 1 4096 4096 4 128
