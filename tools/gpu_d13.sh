for c in 2 4 8; do echo "== C1 cluster=$c"; FLUTE_FORCE_CLUSTER=$c timeout 100 python tools/graph_vs_eager.py 1 4096 4096 4 128; done
for w in 148 222 296; do echo "== W3 workers=$w"; WORKERS=$w timeout 100 python tools/graph_vs_eager.py 1 4096 14336 3 128; done
for w in 148 296; do echo "== W3 M16 workers=$w"; WORKERS=$w timeout 100 python tools/graph_vs_eager.py 16 4096 14336 3 128; done
echo "== W3 14336x4096 stream-k"; FLUTE_NO_CLUSTER=1 timeout 100 python tools/graph_vs_eager.py 1 14336 4096 3 128
echo "== W3 14336x4096 stream-k 296"; WORKERS=296 timeout 100 python tools/graph_vs_eager.py 1 14336 4096 3 128
for c in 2 4; do echo "== W3 14336x4096 cluster=$c"; FLUTE_FORCE_CLUSTER=$c timeout 100 python tools/graph_vs_eager.py 1 14336 4096 3 128; done
