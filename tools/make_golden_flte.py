#!/usr/bin/env python
"""tests/golden/flte.npz: FLTE containers written by the *unmodified reference
library* (quantize_matrix + reorder_and_split + write_flte) for small W2/W3/W4
matrices, with the f32 inputs and the reference's own parse verdicts for a set
of corruptions (section, byte offset).  Run in the build container:

    python tools/make_golden_flte.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import RefLib  # noqa: E402

CASES = [(2, 64, 256, 64), (3, 128, 256, 128), (4, 32, 128, 192)]  # bits, group, k, n


def corruptions(b: bytes):
    """(name, bytes) variants exercising each section of the parser."""
    out = []
    for cut in (0, 3, 4, 5, 6, 10, 14, 18, 19, 25, len(b) - 13, len(b) - 1):
        out.append((f"truncate@{cut}", b[:cut]))
    out.append(("bad_magic", b"FLTX" + b[4:]))
    out.append(("bad_version", b[:4] + bytes([2]) + b[5:]))
    out.append(("bad_bits", b[:5] + bytes([5]) + b[6:]))
    out.append(("bad_slice_count", b[:18] + bytes([3]) + b[19:]))
    out.append(("trailing", b + b"\x00"))
    return out


def main():
    ref = RefLib()
    rng = np.random.default_rng(777)
    blobs, ws, names, secs, offs, meta = [], [], [], [], [], []
    for bits, group, k, n in CASES:
        w = rng.standard_normal((k, n)).astype(np.float32)
        w[:, 0] = 0.0  # zero groups
        b = ref.flte_write(w, bits, group)
        blobs.append(np.frombuffer(b, np.uint8))
        ws.append(w)
        meta.append((bits, group, k, n))
        for name, c in corruptions(b):
            v = ref.flte_parse(c)
            names.append(f"w{bits}:{name}")
            secs.append("" if v is None else v[0])
            offs.append(-1 if v is None else v[1])
    out = {"meta": np.array(meta, np.int64), "names": np.array(names), "sections": np.array(secs),
           "offsets": np.array(offs, np.int64)}
    for i, (bl, w) in enumerate(zip(blobs, ws)):
        out[f"flte{i}"] = bl
        out[f"w{i}"] = w
    np.savez_compressed(os.path.join(ROOT, "tests", "golden", "flte.npz"), **out)
    print("wrote", len(blobs), "containers,", len(names), "corruption verdicts")


if __name__ == "__main__":
    main()
