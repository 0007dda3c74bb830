import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2407_10960_b200 as F
rng = np.random.default_rng(42)
shapes = [(256, 320, 3), (512, 128, 4), (384, 192, 2)]
hs = []
for (k, n, bits) in shapes:
    idx, sc = F.quantize_matrix(rng.standard_normal((k, n)).astype(np.float32), bits, 128)
    hs.append(F.DeviceWeights(idx, sc, F.build_nf_table(bits), bits, 128))
ms=[1, 5, 32, 17, 3, 64]
items, want, host = [], [], []
for i, m in enumerate(ms):
    dw = hs[i % 3]
    x = (rng.standard_normal((m, dw.k)) * 0.5).astype(np.float16)
    want.append(dw.gemm(torch.from_numpy(x).cuda()).cpu().numpy().view(np.uint16))
    host.append(dw.gemm_host(x.view(np.uint16)))
    items.append((dw, x.view(np.uint16), np.zeros((m, dw.n), np.uint16)))
for rep in range(3):
    F.gemm_host_batch(items)
    print("rep", rep, [int((o != w).sum()) for (_, _, o), w in zip(items, want)], "host vs dev", [int((h != w).sum()) for h, w in zip(host, want)])
# single-item batches
for i,(dw,x,o) in enumerate(items):
    o2=np.zeros_like(o); F.gemm_host_batch([(dw,x,o2)]); print("single", i, int((o2!=want[i]).sum()))
