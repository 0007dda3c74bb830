timeout 600 python -m pytest tests/test_gpu_parity.py -q -x --timeout 300 -k "32 or baseline or workers" 2>&1 | tail -2
for cw in 8 12 16; do for c in "32 4096 14336 3 128" "32 14336 4096 3 128" "24 4096 4096 4 128"; do echo "CW$cw $(FLUTE_M32_CW=$cw timeout 60 python tools/graph_vs_eager.py $c)"; done; done 2>&1 | sed 's/R=12 workers=default pdl=on://'
