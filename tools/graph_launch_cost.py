#!/usr/bin/env python
"""Host cost of launching a captured graph of L gemm() calls (PDL on/off via
FLUTE_NO_PDL) and the GPU time of one replay measured with events."""
import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2407_10960_b200 as F
m, k, n, bits, group = 1, 4096, 14336, 3, 128
L = int(sys.argv[1]) if len(sys.argv) > 1 else 48
R = 12
rng = np.random.default_rng(0)
idx, sc = F.quantize_matrix(rng.standard_normal((k, n), dtype=np.float32), bits, group)
dws = [F.DeviceWeights(idx, sc, F.build_nf_table(bits), bits, group) for _ in range(R)]
x = torch.randn(m, k, dtype=torch.float16, device="cuda")
y = torch.empty(m, n, dtype=torch.float16, device="cuda")
st = torch.cuda.Stream()
with torch.cuda.stream(st):
    for i in range(2 * R):
        dws[i % R].gemm(x, y, stream=st.cuda_stream)
st.synchronize()
if os.environ.get("EAGER_FIRST"):
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    with torch.cuda.stream(st):
        e0.record()
        for i in range(L):
            dws[i % R].gemm(x, y, stream=st.cuda_stream)
        e1.record()
    e1.synchronize()
    print(f"eager {e0.elapsed_time(e1) * 1e3 / L:.2f} us/launch")
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=st):
    for i in range(L):
        dws[i % R].gemm(x, y, stream=st.cuda_stream)
for _ in range(3):
    g.replay()
torch.cuda.synchronize()
res = []
for _ in range(5):
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    with torch.cuda.stream(st):
        e0.record()
        t = time.perf_counter()
        g.replay()
        th = time.perf_counter() - t
        e1.record()
    e1.synchronize()
    res.append((th * 1e6, e0.elapsed_time(e1) * 1e3))
    torch.cuda.synchronize()
print(f"L={L} pdl={'off' if os.environ.get('FLUTE_NO_PDL') else 'on'}: host replay() "
      + " ".join(f"{a:.0f}" for a, _ in res) + " us; GPU per replay "
      + " ".join(f"{b:.0f}" for _, b in res) + f" us ({res[-1][1]/L:.2f} us/launch)")

# back-to-back replays: the same graph 6x vs two graph instances alternated
g2 = torch.cuda.CUDAGraph()
with torch.cuda.graph(g2, stream=st):
    for i in range(L):
        dws[i % R].gemm(x, y, stream=st.cuda_stream)
for _ in range(2):
    g2.replay()
torch.cuda.synchronize()
for name, seq in (("same x6", [g] * 6), ("alternating x6", [g, g2] * 3)):
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    with torch.cuda.stream(st):
        e0.record()
        for gg in seq:
            gg.replay()
        e1.record()
    e1.synchronize()
    print(f"  {name}: {e0.elapsed_time(e1) * 1e3 / (6 * L):.2f} us/launch")
