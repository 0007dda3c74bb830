export FLUTE_LIB=paper_2407_10960_b200/libflute_b200_diag.so
for v in 4,8 2,8 8,8 4,16 8,16; do echo "== variant UPS,CW=$v"; FLUTE_VARIANT=$v python tools/perf_cases.py "1 4096 4096 4 128" "1 4096 14336 3 128" "8 4096 14336 3 128"; done
