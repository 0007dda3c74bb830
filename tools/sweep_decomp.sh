# Decomposition sweep: default vs Stream-K 148/296/444 vs forced cluster sizes.
for c in "1 4096 4096 4 128" "1 4096 14336 3 128" "16 4096 14336 3 128" "32 4096 14336 3 128" "1 14336 4096 3 128" "16 14336 4096 3 128" "32 14336 4096 3 128"; do
  echo "### $c"
  timeout 60 python tools/graph_vs_eager.py $c | sed 's/^/default  /'
  for w in 148 296; do WORKERS=$w timeout 60 python tools/graph_vs_eager.py $c | sed "s/^/sk$w  /"; done
  for cl in 1 2 4; do FLUTE_FORCE_CLUSTER=$cl timeout 60 python tools/graph_vs_eager.py $c | sed "s/^/cl$cl  /"; done
done 2>&1 | sed 's/M=[0-9]* K=[0-9]* N=[0-9]* W[0-9]g128 R=12 workers=[a-z0-9]* pdl=on://'
