#!/usr/bin/env python
"""Launch one LUT-GEMM case a few times (no graph) — the target for
`ncu --set full` captures and launch lists.  Also prints per-launch CUDA-event
timings (with L2 rotation) when run without a profiler.

usage: python tools/profile_case.py M K N BITS GROUP [launches] [workers]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2407_10960_b200 as F  # noqa: E402


def main():
    m, k, n, bits, group = (int(v) for v in sys.argv[1:6])
    launches = int(sys.argv[6]) if len(sys.argv) > 6 else 8
    workers = int(sys.argv[7]) if len(sys.argv) > 7 else 0
    rng = np.random.default_rng(0)
    idx, scales = F.quantize_matrix(rng.standard_normal((k, n), dtype=np.float32), bits, group)
    table = F.build_nf_table(bits)
    reps = max(2, int(np.ceil(3 * 126e6 / F.algorithmic_bytes(m, k, n, bits, group))))
    reps = min(reps, 64)
    dws = [F.DeviceWeights(idx, scales, table, bits, group) for _ in range(reps)]
    x = torch.randn(m, k, dtype=torch.float16, device="cuda") * 0.5
    y = torch.empty(m, n, dtype=torch.float16, device="cuda")
    for i in range(launches):
        dws[i % reps].gemm(x, y, workers=workers)
    torch.cuda.synchronize()
    if os.environ.get("NCU_PROFILING") or "NV_COMPUTE_PROFILER" in os.environ:
        return
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(200):
        dws[i % reps].gemm(x, y, workers=workers)
    e1.record()
    e1.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / 200
    b = F.algorithmic_bytes(m, k, n, bits, group)
    print(f"M={m} K={k} N={n} W{bits}g{group}: {us:.2f} us/launch (eager, incl. launch gaps), "
          f"{b / us / 1e3:.0f} GB/s")


if __name__ == "__main__":
    main()
