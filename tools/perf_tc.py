#!/usr/bin/env python
"""Compute-bound regime (BASELINE configs[4]): W4 g128 M=64..512 via the
tcgen05 path vs cuBLAS fp16 of the same shape; CUDA-graph timings with weight
replicas rotated.  usage: python tools/perf_tc.py [K N] ..."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.environ.get("PKGROOT") or os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2407_10960_b200 as F  # noqa: E402


def gtime(fn, reps=20):
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        for _ in range(8):  # every replica once (workspace growth happens outside capture)
            fn()
    st.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        for _ in range(reps):
            fn()
    with torch.cuda.stream(st):
        g.replay()
    torch.cuda.synchronize()  # the warm replay must not overlap the timed ones
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    with torch.cuda.stream(st):
        e0.record()
        for _ in range(5):
            g.replay()
        e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) * 1e3 / (5 * reps)


def main():
    shapes = [(4096, 4096), (8192, 8192)]
    if len(sys.argv) > 2:
        shapes = [(int(sys.argv[1]), int(sys.argv[2]))]
    for (k, n) in shapes:
        rng = np.random.default_rng(k + n)
        idx, sc = F.quantize_matrix(rng.standard_normal((k, n), dtype=np.float32), 4, 128)
        R = 4
        dws = [F.DeviceWeights(idx, sc, F.build_nf_table(4), 4, 128) for _ in range(R)]
        wd = [torch.randn(k, n, dtype=torch.float16, device="cuda") for _ in range(R)]
        for m in (64, 128, 256, 512):
            x = torch.randn(m, k, dtype=torch.float16, device="cuda")
            y = torch.empty(m, n, dtype=torch.float16, device="cuda")
            cnt = [0]

            def ours():
                dws[cnt[0] % R].gemm(x, y)
                cnt[0] += 1

            def cub():
                torch.matmul(x, wd[cnt[0] % R], out=y)
                cnt[0] += 1
            t_ours = gtime(ours)
            t_cub = gtime(cub)
            fl = 2 * m * k * n
            print(f"M={m:4d} K={k} N={n} W4g128: ours {t_ours:7.2f} us {fl / t_ours / 1e6:7.1f} TFLOP/s"
                  f" | cuBLAS fp16 {t_cub:7.2f} us {fl / t_cub / 1e6:7.1f} TFLOP/s | x{t_cub / t_ours:.2f}",
                  flush=True)


if __name__ == "__main__":
    main()
