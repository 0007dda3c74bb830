#!/usr/bin/env python
"""Per-CTA timeline of one qgemm launch (diag build: FLUTE_DEBUG_TIMES).

usage: python tools/timeline.py M K N BITS GROUP [workers] [--stages]
Prints, per stamp, min / median / max over CTAs in µs relative to the earliest
CTA start; with --stages also the per-stage trace of consumer warp 0 of CTAs
0 and 74 (wait begin -> data ready -> compute done).
"""
import os
import sys

os.environ["FLUTE_DEBUG_TIMES"] = "1"
_ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.environ.setdefault("FLUTE_LIB", os.path.join(_ROOT, "paper_2407_10960_b200",
                                                "libflute_b200_diag.so"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

sys.path.insert(0, _ROOT)
import paper_2407_10960_b200 as F  # noqa: E402

NAMES = ["start", "producer_issued", "lut_ready", "first_stage", "seg_end", "last_seg_end", "exit",
         "finisher_acq", "cta_barrier", "prod_policy", "prod_pdl_wait", "lut_filled", "epi_pdl_wait"]


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    show_stages = "--stages" in sys.argv
    m, k, n, bits, group = (int(v) for v in args[:5])
    workers = int(args[5]) if len(args) > 5 else 0
    rng = np.random.default_rng(0)
    idx, scales = F.quantize_matrix(rng.standard_normal((k, n), dtype=np.float32), bits, group)
    reps = 6
    dws = [F.DeviceWeights(idx, scales, F.build_nf_table(bits), bits, group) for _ in range(reps)]
    x = torch.randn(m, k, dtype=torch.float16, device="cuda")
    y = torch.empty(m, n, dtype=torch.float16, device="cuda")
    P = workers or F.default_workers(m, k, n, bits)
    for i in range(reps):
        dws[i].gemm(x, y, workers=workers)
        torch.cuda.synchronize()
    t, tr = F.debug_times(P)
    t = t.astype(np.int64)
    t0 = t[:, 0][t[:, 0] > 0].min()
    rel = np.where(t > 0, (t - t0) / 1e3, np.nan)
    print(f"M={m} K={k} N={n} W{bits}g{group} P={P}")
    for j, nm in enumerate(NAMES):
        col = rel[:, j]
        col = col[~np.isnan(col)]
        if col.size:
            print(f"  {nm:16s} min {col.min():8.2f}  med {np.median(col):8.2f}  "
                  f"max {col.max():8.2f} us  (n={col.size})")
    if show_stages:
        for cta in (0, P // 2):
            rows = tr[cta].astype(np.int64)
            rows = rows[rows[:, 0] > 0]
            print(f"  CTA {cta}: stage  wait_begin  ready  done   (us; wait, compute)")
            for i, (a, b, c) in enumerate(rows):
                print(f"    {i:3d} {(a - t0) / 1e3:8.2f} {(b - t0) / 1e3:8.2f} {(c - t0) / 1e3:8.2f}"
                      f"   ({(b - a) / 1e3:5.2f}, {(c - b) / 1e3:5.2f})")


if __name__ == "__main__":
    main()
