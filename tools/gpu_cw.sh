timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharding.py -q -x --timeout 300 2>&1 | tail -2
for c in "1 4096 4096 4 128" "16 4096 4096 4 128" "1 4096 14336 3 128" "4 4096 14336 3 128" "16 4096 14336 3 128" "1 14336 4096 3 128" "16 14336 4096 3 128" "1 8192 8192 2 128"; do
  echo "CW16 $(timeout 60 python tools/graph_vs_eager.py $c)"
  echo "CW8  $(FLUTE_CW8=1 timeout 60 python tools/graph_vs_eager.py $c)"
done 2>&1 | sed 's/R=12 workers=default pdl=on://'
