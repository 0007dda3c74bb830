O=gpurun_out/d2; mkdir -p $O
( timeout 200 tools/_build/pdl_stream_bench
export FLUTE_LIB=paper_2407_10960_b200/libflute_b200_diag.so
for v in 1 2 4; do for c in "1 4096 4096 4 128" "1 4096 14336 3 128"; do echo "== UPS=$v $c"; FLUTE_VARIANT=$v timeout 100 python tools/graph_vs_eager.py $c; done; done
) > $O/out.txt 2>&1; cat $O/out.txt
