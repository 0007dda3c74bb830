#!/usr/bin/env python
"""Generate tests/golden/*.npz from the *unmodified reference library*
(oracle/_ref/libflutesim_ref.so, compiled from /root/reference by
oracle/Makefile).  Run in the build container (the reference does not exist on
the GPU box); the fixtures are committed so tests can pin the oracle anywhere.

    python tools/make_golden.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import RefLib  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")
LAYOUTS = [(16, 64, 64, 16, 8, 16), (16, 32, 32, 16, 8, 16), (16, 16, 32, 16, 8, 16),
           (16, 16, 16, 16, 8, 16)]


def main():
    os.makedirs(OUT, exist_ok=True)
    ref = RefLib()
    rng = np.random.default_rng(20240715)

    # numerics: random binary32 patterns + values in the half range
    raw = rng.integers(0, 2 ** 32, 6000, dtype=np.uint64).astype(np.uint32)
    raw = raw[~np.isnan(raw.view(np.float32))]
    vals = np.concatenate([raw.view(np.float32), rng.uniform(-7e4, 7e4, 2000).astype(np.float32),
                           rng.uniform(-1e-4, 1e-4, 2000).astype(np.float32)])
    f16 = np.array([ref.f32_to_f16(v) for v in vals], np.uint16)
    np.savez_compressed(os.path.join(OUT, "numerics.npz"), f32=vals, f16=f16)

    # NF tables
    np.savez_compressed(os.path.join(OUT, "nf_tables.npz"),
                        **{f"nf{b}": ref.nf_table(b) for b in (2, 3, 4)})

    # quantize + pack + vLUT
    qp = {}
    for bits in (2, 3, 4):
        for group in (32, 64):
            w = rng.standard_normal((128, 64)).astype(np.float32)
            w[:group, 5] = 0.0  # an all-zero group -> zero index, scale 0
            idx, sc = ref.quantize(w, bits, group)
            key = f"b{bits}g{group}"
            qp[f"{key}_w"] = w
            qp[f"{key}_idx"] = idx
            qp[f"{key}_scales"] = sc
            for li, L in enumerate(LAYOUTS):
                sl = ref.pack(idx, bits, L)
                for si, s in enumerate(sl):
                    qp[f"{key}_L{li}_s{si}"] = s
        qp[f"vlut{bits}"] = ref.vlut(ref.nf_table(bits), bits)
    qp["layouts"] = np.array(LAYOUTS, np.int32)
    np.savez_compressed(os.path.join(OUT, "quant_pack.npz"), **qp)

    # Stream-K plans (grids from test_streamk.cpp + device-scale grids)
    sk = {}
    grids = [(5, 7, 1, 3), (2, 3, 4, 1), (2, 2, 3, 12), (1, 2, 1, 5), (3, 5, 7, 16), (1, 7, 4, 3),
             (1, 64, 64, 148), (1, 224, 32, 148), (2, 64, 32, 296)]
    for (tm, tn, tk, P) in grids:
        r, f, slots = ref.plan_stream_k(tm, tn, tk, P)
        key = f"g{tm}_{tn}_{tk}_{P}"
        sk[key + "_ranges"] = r
        sk[key + "_fixups"] = f
        sk[key + "_slots"] = np.array([slots], np.int64)
    np.savez_compressed(os.path.join(OUT, "streamk.npz"), **sk)

    # engine: reference execute outputs + TrafficStats at small shapes
    ex = {}
    cases = [(3, 256, 128, 4, 128, 1), (3, 256, 128, 4, 128, 3), (5, 256, 128, 3, 64, 8),
             (1, 512, 256, 3, 128, 16), (17, 256, 64, 2, 32, 2), (4, 128, 64, 4, 32, 7)]
    for ci, (m, k, n, bits, group, P) in enumerate(cases):
        w = rng.standard_normal((k, n)).astype(np.float32)
        idx, sc = ref.quantize(w, bits, group)
        x16 = (rng.standard_normal((m, k)) * 0.5).astype(np.float16).view(np.uint16)
        table = ref.nf_table(bits)
        sl = ref.pack(idx, bits)
        y, st = ref.execute(x16, sl, k, n, bits, group, sc, table, workers=P)
        pt = ref.plan_traffic(m, k, n, bits, group, workers=P)
        ex[f"c{ci}_meta"] = np.array([m, k, n, bits, group, P], np.int64)
        ex[f"c{ci}_idx"] = idx
        ex[f"c{ci}_scales"] = sc
        ex[f"c{ci}_x16"] = x16
        ex[f"c{ci}_y16"] = y
        ex[f"c{ci}_stats"] = st
        ex[f"c{ci}_plan_traffic"] = pt
    np.savez_compressed(os.path.join(OUT, "engine.npz"), **ex)
    for f in sorted(os.listdir(OUT)):
        print(f, os.path.getsize(os.path.join(OUT, f)))


if __name__ == "__main__":
    main()
