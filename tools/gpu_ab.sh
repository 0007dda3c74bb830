for c in "32 4096 14336 3 128" "1 4096 14336 3 128" "16 4096 14336 3 128"; do
  echo "### $c"
  timeout 60 python tools/graph_vs_eager.py $c | sed 's/^/HEAD     /'
  for v in af9a2fe bc9aa38; do PKGROOT=tools/_build/pkg_$v timeout 60 python tools/graph_vs_eager.py $c | sed "s/^/$v  /"; done
done 2>&1 | sed 's/M=[0-9]* K=[0-9]* N=[0-9]* W[0-9]g128 R=12 workers=[a-z0-9]* pdl=on://'
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv
