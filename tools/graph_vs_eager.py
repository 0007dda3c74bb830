#!/usr/bin/env python
"""Per-launch time of one case: eager launches vs a captured CUDA graph, with
R weight replicas rotated (R large = cold HBM).  usage: M K N BITS GROUP [R]"""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.environ.get("PKGROOT") or os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2407_10960_b200 as F

m, k, n, bits, group = (int(v) for v in sys.argv[1:6])
R = int(sys.argv[6]) if len(sys.argv) > 6 else 12
rng = np.random.default_rng(0)
idx, sc = F.quantize_matrix(rng.standard_normal((k, n), dtype=np.float32), bits, group)
dws = [F.DeviceWeights(idx, sc, F.build_nf_table(bits), bits, group) for _ in range(R)]
x = torch.randn(m, k, dtype=torch.float16, device="cuda")
y = torch.empty(m, n, dtype=torch.float16, device="cuda")
st = torch.cuda.Stream()
W = int(os.environ.get("WORKERS", "0"))
def run(n_launch):
    for i in range(n_launch):
        dws[i % R].gemm(x, y, workers=W, stream=st.cuda_stream)
with torch.cuda.stream(st):
    run(2 * R)
st.synchronize()
def timeit(fn, reps):
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    with torch.cuda.stream(st):
        e0.record(); fn(); e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) * 1e3 / reps
L = int(os.environ.get("GL", "4")) * R
eager = timeit(lambda: run(L), L)
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=st):
    run(L)
with torch.cuda.stream(st):
    g.replay()
torch.cuda.synchronize()  # the warm replay must not overlap the timed ones
graph = timeit(lambda: [g.replay() for _ in range(5)], 5 * L)
b = F.algorithmic_bytes(m, k, n, bits, group)
print(f"M={m} K={k} N={n} W{bits}g{group} R={R} workers={W or 'default'} pdl={'off' if os.environ.get('FLUTE_NO_PDL') else 'on'}: "
      f"eager {eager:.2f} us ({b/eager/1e3:.0f} GB/s)  graph {graph:.2f} us ({b/graph/1e3:.0f} GB/s)")
