#!/usr/bin/env python
"""Per-CTA timeline of one qgemm launch (FLUTE_DEBUG_TIMES instrumentation).

usage: python tools/timeline.py M K N BITS GROUP [workers]
Prints, per stamp, min / median / max over CTAs in µs relative to the earliest
CTA start: start, producer issued, LUT ready, first stage landed, segment end,
last segment end, exit.
"""
import os
import sys

os.environ["FLUTE_DEBUG_TIMES"] = "1"
import numpy as np  # noqa: E402
import torch  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2407_10960_b200 as F  # noqa: E402

NAMES = ["start", "producer_issued", "lut_ready", "first_stage", "seg_end", "last_seg_end", "exit"]


def main():
    m, k, n, bits, group = (int(v) for v in sys.argv[1:6])
    workers = int(sys.argv[6]) if len(sys.argv) > 6 else 0
    rng = np.random.default_rng(0)
    idx, scales = F.quantize_matrix(rng.standard_normal((k, n), dtype=np.float32), bits, group)
    reps = 8
    dws = [F.DeviceWeights(idx, scales, F.build_nf_table(bits), bits, group) for _ in range(reps)]
    x = torch.randn(m, k, dtype=torch.float16, device="cuda")
    y = torch.empty(m, n, dtype=torch.float16, device="cuda")
    P = workers or F.default_workers(m, k, n, bits)
    for i in range(reps):
        dws[i].gemm(x, y, workers=workers)
        torch.cuda.synchronize()
        t = F.debug_times(P).astype(np.int64)
        t0 = t[:, 0][t[:, 0] > 0].min()
        rel = np.where(t > 0, (t - t0) / 1e3, np.nan)
        if i >= reps - 2:
            print(f"launch {i}: M={m} K={k} N={n} W{bits}g{group} P={P}")
            for j, nm in enumerate(NAMES):
                col = rel[:, j]
                col = col[~np.isnan(col)]
                if col.size:
                    print(f"  {nm:16s} min {col.min():8.2f}  med {np.median(col):8.2f}  "
                          f"max {col.max():8.2f} us  (n={col.size})")


if __name__ == "__main__":
    main()
