export FLUTE_LIB=paper_2407_10960_b200/libflute_b200_diag.so
for c in "1 4096 14336 3 128" "1 4096 4096 4 128"; do echo "== timeline $c"; timeout 100 python tools/timeline.py $c --stages; done
for c in "1 4096 14336 3 128" "1 4096 4096 4 128"; do echo "== NO_PDL $c"; FLUTE_NO_PDL=1 timeout 100 python tools/graph_vs_eager.py $c; done
