#!/usr/bin/env python
"""Where the end-to-end step time goes: one HostBatch replay of the bench
workload timed by wall clock and by CUDA events on the launching stream, and
the same GEMMs with device-resident inputs (no copies) for comparison."""
import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2407_10960_b200 as F
MS, SHAPES = (1, 4, 16, 32), ((4096, 14336), (14336, 4096))
rng = np.random.default_rng(0)
W = {}
for (k, n) in SHAPES:
    idx, sc = F.quantize_matrix(rng.standard_normal((k, n), dtype=np.float32), 3, 128)
    W[(k, n)] = [F.DeviceWeights(idx, sc, F.build_nf_table(3), 3, 128) for _ in range(3)]
cases = [(m, k, n) for m in MS for (k, n) in SHAPES]
xp = {(m, k): torch.randn(m, k, dtype=torch.float16).pin_memory() for (m, k, n) in cases}
yp = {(m, n): torch.empty(m, n, dtype=torch.float16).pin_memory() for (m, k, n) in cases}
xd = {key: t.cuda() for key, t in xp.items()}
yd = {key: t.cuda() for key, t in yp.items()}
st = torch.cuda.Stream()
GRAPH = os.environ.get("EAGER") is None
batches = [F.HostBatch([(W[(k, n)][r], xp[(m, k)].numpy().view(np.uint16), yp[(m, n)].numpy().view(np.uint16))
                        for (m, k, n) in cases], graph=GRAPH) for r in range(3)]
for _ in range(5):
    for b in batches:
        b.run(st.cuda_stream)
walls, evs = [], []
for it in range(30):
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    with torch.cuda.stream(st):
        e0.record()
    t = time.perf_counter()
    batches[it % 3].run(st.cuda_stream)
    walls.append((time.perf_counter() - t) * 1e6)
    with torch.cuda.stream(st):
        e1.record()
    e1.synchronize()
    evs.append(e0.elapsed_time(e1) * 1e3)
# device-resident, same GEMMs, eager
with torch.cuda.stream(st):
    for _ in range(3):
        for r in range(3):
            for (m, k, n) in cases:
                W[(k, n)][r].gemm(xd[(m, k)], yd[(m, n)], stream=st.cuda_stream)
st.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
with torch.cuda.stream(st):
    e0.record()
    for it in range(30):
        for (m, k, n) in cases:
            W[(k, n)][it % 3].gemm(xd[(m, k)], yd[(m, n)], stream=st.cuda_stream)
    e1.record()
e1.synchronize()
print(f"{'graph' if GRAPH else 'eager'} HostBatch step: wall median {np.median(walls):.1f} us, events median {np.median(evs):.1f} us; "
      f"device-resident GEMMs only {e0.elapsed_time(e1) * 1e3 / 30:.1f} us/step")
