for w in 0 296 444; do for c in "1 4096 4096 4 128" "1 4096 14336 3 128" "16 4096 14336 3 128"; do WORKERS=$w timeout 100 python tools/graph_vs_eager.py $c; done; done
