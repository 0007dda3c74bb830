#!/usr/bin/env python
"""Steady-state timeline: N back-to-back launches (PDL, no sync, distinct weight
replicas) with per-CTA stamps for each (diag build, FLUTE_DEBUG_TIMES=N ring).
usage: python tools/timeline_ring.py M K N BITS GROUP [launches]"""
import os
import sys

_ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
L = int(sys.argv[6]) if len(sys.argv) > 6 else 6
os.environ["FLUTE_DEBUG_TIMES"] = str(L)
os.environ.setdefault("FLUTE_LIB", os.path.join(_ROOT, "paper_2407_10960_b200", "libflute_b200_diag.so"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

sys.path.insert(0, _ROOT)
import paper_2407_10960_b200 as F  # noqa: E402

NAMES = ["start", "producer_issued", "lut_ready", "first_stage", "seg_end", "last_seg_end", "exit",
         "finisher_acq", "cta_barrier", "prod_policy", "prod_pdl_wait", "lut_filled", "epi_pdl_wait"]


def main():
    m, k, n, bits, group = (int(v) for v in sys.argv[1:6])
    rng = np.random.default_rng(0)
    idx, sc = F.quantize_matrix(rng.standard_normal((k, n), dtype=np.float32), bits, group)
    dws = [F.DeviceWeights(idx, sc, F.build_nf_table(bits), bits, group) for _ in range(L)]
    x = torch.randn(m, k, dtype=torch.float16, device="cuda")
    y = torch.empty(m, n, dtype=torch.float16, device="cuda")
    W = int(os.environ.get("WORKERS", "0"))
    P = W or F.default_workers(m, k, n, bits)
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        for i in range(L):  # warm (fills the ring once)
            dws[i].gemm(x, y, workers=W, stream=st.cuda_stream)
    st.synchronize()
    if os.environ.get("GRAPH"):  # same launches captured into a CUDA graph and replayed
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for i in range(L):
                dws[i].gemm(x, y, workers=W, stream=st.cuda_stream)
        g.replay()
        st.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        with torch.cuda.stream(st):
            e0.record()
            g.replay()
            e1.record()
        e1.synchronize()
        print(f"events around one replay: {e0.elapsed_time(e1) * 1e3 / L:.2f} us per launch")
    else:
        with torch.cuda.stream(st):
            for i in range(L):
                dws[i].gemm(x, y, workers=W, stream=st.cuda_stream)
    st.synchronize()
    res = F.debug_times(P, L)
    t0 = min(int(r[0][:, 0][r[0][:, 0] > 0].min()) for r in res)
    print(f"M={m} K={k} N={n} W{bits}g{group} P={P}, {L} back-to-back launches (us from first start)")
    print("launch " + " ".join(f"{nm[:12]:>12s}" for nm in ["start", "prod_pdl_wait", "last_seg_end", "cons_exit", "epi_done(max)"]))
    for i, (stamps, _) in enumerate(res):
        t = stamps.astype(np.int64)
        def col(j, f):
            c = t[:, j]
            c = c[c > 0]
            return (f(c) - t0) / 1e3 if c.size else float("nan")
        print(f"{i:6d} " + " ".join(f"{v:12.2f}" for v in
                                    [col(0, np.min), col(10, np.median),
                                     col(5, np.max), col(6, np.max), col(15, np.max)]))


    # CTA placement: CTAs per SM of the last launch (diag slot 13 = %smid)
    sm = res[-1][0].astype(np.int64)[:P, 13]
    counts = np.bincount(sm, minlength=148)
    hist = np.bincount(counts)
    print("CTAs per SM (last launch): " + ", ".join(f"{c} CTAs: {h} SMs" for c, h in enumerate(hist) if h))
    exits = []
    for stamps, _ in res:
        c = stamps.astype(np.int64)[:, 6]
        exits.append(c[c > 0].max())
    if L > 3:
        print(f"steady state: {(exits[-1] - exits[1]) / (L - 2) / 1e3:.2f} us per launch "
              f"(last-CTA exit to last-CTA exit, launches 1..{L - 1})")

    if os.environ.get("STAGES"):
        stamps, tr = res[min(3, L - 1)]
        for cta in (0, P // 2, P - 1):
            rows = tr[cta].astype(np.int64)
            rows = rows[rows[:, 0] > 0]
            print(f"  launch {min(3, L - 1)} CTA {cta}: wait_begin ready done (us; wait, compute)")
            for i, (a, b, c) in enumerate(rows):
                print(f"    {i:3d} {(a - t0) / 1e3:8.2f} {(b - t0) / 1e3:8.2f} {(c - t0) / 1e3:8.2f}"
                      f"   ({(b - a) / 1e3:5.2f}, {(c - b) / 1e3:5.2f})")


if __name__ == "__main__":
    main()
