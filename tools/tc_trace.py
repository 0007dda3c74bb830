#!/usr/bin/env python
"""Timeline of one tcgen05-kernel launch (diag build, FLUTE_TC_TRACE).
usage: FLUTE_LIB=paper_2407_10960_b200/libflute_b200_diag.so python tools/tc_trace.py M K N BITS GROUP"""
import os
import sys
import tempfile

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("FLUTE_LIB", os.path.join(ROOT, "paper_2407_10960_b200", "libflute_b200_diag.so"))
path = os.path.join(tempfile.gettempdir(), "flute_tc_trace.bin")
import paper_2407_10960_b200 as F  # noqa: E402

m, k, n, bits, group = (int(v) for v in sys.argv[1:6])
rng = np.random.default_rng(0)
idx, sc = F.quantize_matrix(rng.standard_normal((k, n), dtype=np.float32), bits, group)
dws = [F.DeviceWeights(idx, sc, F.build_nf_table(bits), bits, group) for _ in range(4)]
x = torch.randn(m, k, dtype=torch.float16, device="cuda")
for i in range(3):
    dws[i].gemm(x)
torch.cuda.synchronize()
os.environ["FLUTE_TC_TRACE"] = path
dws[3].gemm(x)
torch.cuda.synchronize()
raw = np.fromfile(path, np.uint64)
ctas, st = int(raw[0]), int(raw[1])
cta = raw[2:2 + ctas * 4].reshape(ctas, 4).astype(np.int64)
stg = raw[2 + ctas * 4:].reshape(ctas, st, 8).astype(np.int64)
t0 = cta[:, 0][cta[:, 0] > 0].min()
rel = lambda v: (v - t0) / 1e3
print(f"M={m} K={k} N={n} W{bits}g{group}: {ctas} CTAs")
print(f"  CTA start   min {rel(cta[:,0].min()):7.2f}  med {rel(np.median(cta[:,0])):7.2f}  max {rel(cta[:,0].max()):7.2f} us")
print(f"  acc_full    min {rel(cta[:,1].min()):7.2f}  med {rel(np.median(cta[:,1])):7.2f}  max {rel(cta[:,1].max()):7.2f} us")
print(f"  X pdl_wait  min {rel(cta[:,3].min()):7.2f}  med {rel(np.median(cta[:,3])):7.2f}  max {rel(cta[:,3].max()):7.2f} us")
print(f"  epilogue    min {rel(cta[:,2].min()):7.2f}  med {rel(np.median(cta[:,2])):7.2f}  max {rel(cta[:,2].max()):7.2f} us")
for c in (0, ctas // 2, ctas - 1):
    print(f"  CTA {c}: stage  w_full  loads_done a_empty  stores_issued st_waited a_full  mma_ready   (us)")
    for i in range(st):
        r = stg[c, i]
        if r[0] == 0:
            break
        print(f"    {i:3d} {rel(r[0]):8.2f} {rel(r[6]):8.2f} {rel(r[1]):8.2f} {rel(r[4]):8.2f} {rel(r[5]):8.2f} {rel(r[2]):8.2f}   mma: a_full seen {rel(r[7]):8.2f} x_full seen {rel(r[3]):8.2f}")
