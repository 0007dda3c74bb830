#!/usr/bin/env python
"""Quick per-case timing in ONE process (keeps GPU calls short): back-to-back
eager launches (PDL on) rotating weight replicas so weights stream from HBM.

usage: python tools/perf_cases.py "M K N BITS GROUP" ["M K N BITS GROUP" ...]
       (no args: the BASELINE headline cases)
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2407_10960_b200 as F  # noqa: E402

DEFAULT = ["1 4096 4096 4 128", "16 4096 4096 4 128", "1 4096 14336 3 128",
           "4 4096 14336 3 128", "16 4096 14336 3 128", "32 4096 14336 3 128",
           "1 14336 4096 3 128", "32 14336 4096 3 128"]


def main():
    cases = sys.argv[1:] or DEFAULT
    st = torch.cuda.Stream()
    cache = {}
    for c in cases:
        m, k, n, bits, group = (int(v) for v in c.split())
        key = (k, n, bits, group)
        if key not in cache:
            rng = np.random.default_rng(k + n + bits)
            w = rng.standard_normal((k, n), dtype=np.float32)
            idx, sc = F.quantize_matrix(w, bits, group)
            R = max(2, min(8, int(np.ceil(2.5 * 126e6 / F.algorithmic_bytes(1, k, n, bits, group)))))
            cache[key] = [F.DeviceWeights(idx, sc, F.build_nf_table(bits), bits, group)
                          for _ in range(R)]
        dws = cache[key]
        R = len(dws)
        x = torch.randn(m, k, dtype=torch.float16, device="cuda")
        y = torch.empty(m, n, dtype=torch.float16, device="cuda")
        with torch.cuda.stream(st):
            for i in range(2 * R):
                dws[i % R].gemm(x, y, stream=st.cuda_stream)
        st.synchronize()
        L = 20 * R
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        with torch.cuda.stream(st):
            e0.record()
            for i in range(L):
                dws[i % R].gemm(x, y, stream=st.cuda_stream)
            e1.record()
        e1.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / L
        b = F.algorithmic_bytes(m, k, n, bits, group)
        print(f"M={m:3d} K={k:6d} N={n:6d} W{bits}g{group}: {us:7.2f} us  {b / us / 1e3:6.0f} GB/s",
              flush=True)


if __name__ == "__main__":
    main()
