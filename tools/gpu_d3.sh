export FLUTE_LIB=paper_2407_10960_b200/libflute_b200_diag.so
for d in 0 1 15; do for c in "1 4096 4096 4 128" "1 4096 14336 3 128"; do echo "== DIAG=$d"; FLUTE_DIAG=$d timeout 100 python tools/graph_vs_eager.py $c; done; done
for c in "1 4096 4096 4 128" "1 4096 14336 3 128"; do echo "== DIAG=15 timeline $c"; FLUTE_DIAG=15 timeout 100 python tools/timeline.py $c; done
echo "== workers=1 DIAG=15"; WORKERS=1 FLUTE_DIAG=15 timeout 100 python tools/graph_vs_eager.py 1 4096 4096 4 128
echo "== workers=8 DIAG=15"; WORKERS=8 FLUTE_DIAG=15 timeout 100 python tools/graph_vs_eager.py 1 4096 4096 4 128
echo "== workers=64 DIAG=15"; WORKERS=64 FLUTE_DIAG=15 timeout 100 python tools/graph_vs_eager.py 1 4096 4096 4 128
echo "== workers=64 DIAG=0"; WORKERS=64 timeout 100 python tools/graph_vs_eager.py 1 4096 4096 4 128
echo "== workers=128 DIAG=0"; WORKERS=128 timeout 100 python tools/graph_vs_eager.py 1 4096 4096 4 128
