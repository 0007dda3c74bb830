for c in "1 4096 4096 4 128" "1 4096 14336 3 128" "16 4096 14336 3 128" "32 4096 14336 3 128" "1 14336 4096 3 128"; do
  echo "### $c"
  timeout 60 python tools/graph_vs_eager.py $c | sed 's/^/sleep-all  /'
  FLUTE_LIB=tools/_build/lib_nsp.so timeout 60 python tools/graph_vs_eager.py $c | sed 's/^/sleep-epi  /'
  PKGROOT=tools/_build/pkg_af9a2fe timeout 60 python tools/graph_vs_eager.py $c | sed "s/^/af9a2fe    /"
done 2>&1 | sed 's/M=[0-9]* K=[0-9]* N=[0-9]* W[0-9]g128 R=12 workers=[a-z0-9]* pdl=on://'
