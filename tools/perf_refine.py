#!/usr/bin/env python
"""Learned-sigma refinement (§8(f) row 3): one ste_evaluate on the GPU vs the
reference library's OpenMP CPU ste_evaluate, same inputs; checks the GPU
gradients are bit-identical.  usage: python tools/perf_refine.py [K N M]"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402  (checker + CPU baseline only)
import paper_2407_10960_b200 as F  # noqa: E402

k, n, m = (int(v) for v in sys.argv[1:4]) if len(sys.argv) > 3 else (4096, 4096, 128)
rng = np.random.default_rng(0)
w = (rng.standard_t(3, (k, n)) * 0.02).astype(np.float32)
x = rng.standard_normal((m, k)).astype(np.float32)
s = np.full(k // 128 * n, F.nf_sigma())
F.ste_evaluate(w[:256, :64], x[:, :256], 4, 128, s[:2 * 64])  # context warm-up
t = time.perf_counter()
lg, gg, ig = F.ste_evaluate(w, x, 4, 128, s)
tg = time.perf_counter() - t
ref = oracle.RefLib() if oracle.RefLib.available() else oracle.Oracle()
t = time.perf_counter()
lr, gr, ir = ref.ste_evaluate(w, x, 4, 128, s)
tc = time.perf_counter() - t
flop = 2 * 2.0 * m * k * n
print(f"ste_evaluate K={k} N={n} M={m} W4g128: GPU {tg*1e3:.1f} ms (incl. H2D of W/X, "
      f"{flop/tg/1e12:.2f} TFLOP/s f64 eff.) | CPU {type(ref).__name__} {tc*1e3:.0f} ms "
      f"({os.cpu_count()} cores) | x{tc/tg:.0f} | grads bit-identical: {np.array_equal(gg, gr)}, "
      f"indices: {np.array_equal(ig, ir)}, loss rel diff {abs(lg-lr)/abs(lr):.1e}")
