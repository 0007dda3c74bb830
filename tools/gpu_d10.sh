export FLUTE_LIB=paper_2407_10960_b200/libflute_b200_diag.so
for d in 0 15 31 47 63 127 1 17 113; do echo "== DIAG=$d"; FLUTE_DIAG=$d timeout 100 python tools/graph_vs_eager.py 1 4096 4096 4 128; done
for d in 0 16; do echo "== W3 DIAG=$d"; FLUTE_DIAG=$d timeout 100 python tools/graph_vs_eager.py 1 4096 14336 3 128; done
