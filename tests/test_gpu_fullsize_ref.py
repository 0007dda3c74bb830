"""Full BASELINE-size parity against the reference engine's OWN output.

SURVEY.md §8(c)(ii): at configs[0] (W4 g128 4096x4096) and configs[1] (W3
g128 LLaMA-3-8B MLP shapes) the CUDA path is compared per element with both
  * y64   — binary64 product over the f16-rounded dequantised weights, and
  * y_ref — flutesim::execute of the UNMODIFIED reference library
            (oracle/_ref, engine.cpp:345-373) at P = host cores,
with the bound |y - z| <= 1e-2 * max(|z|, rms(z)) (north_star tolerance,
written here).  Reported per case (FLUTE_PARITY_REPORT=path appends one JSON
line): max |y - y_ref| in f16 ulps, ||y - y_ref||_2 / ||y_ref||_2, the same
against y64, and the reference's own distance to y64 for comparison.
Reference test this extends: test_engine.cpp:141-160 (binary64 sweep, which
stops at K = 512).
"""
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL = 1e-2

CASES = [(m, 4096, 4096, 4, 128) for m in (1, 4, 16)] + \
        [(m, k, n, 3, 128) for m in (1, 4, 16, 32) for (k, n) in ((4096, 14336), (14336, 4096))]


def _ulp_diff(a16, b16):
    """|a - b| in binary16 ulps (ordered-integer distance of the bit patterns)."""
    def ordered(u):
        u = u.astype(np.int32)
        return np.where(u & 0x8000, 0x8000 - (u & 0x7FFF), 0x8000 + u)
    return np.abs(ordered(a16) - ordered(b16))


def _bound_ok(y, z, tol=TOL):
    bound = tol * np.maximum(np.abs(z), np.sqrt(np.mean(z ** 2)) + 1e-30)
    err = np.abs(y - z)
    return bool(np.all(err <= bound)), float((err / bound).max())


@pytest.mark.parametrize("m,k,n,bits,group", CASES)
def test_fullsize_vs_reference_engine(F, orc, ref, gpu, m, k, n, bits, group):
    rng = np.random.default_rng(2407 + m + k + bits)
    w = rng.standard_normal((k, n), dtype=np.float32)
    idx, scales = ref.quantize(w, bits, group)       # the reference's own quantizer
    table = ref.nf_table(bits)
    x16 = (rng.standard_normal((m, k)) * 0.5).astype(np.float16).view(np.uint16)

    dw = F.DeviceWeights(idx, scales, table, bits, group)
    y16 = dw.gemm(gpu.from_numpy(x16.view(np.float16)).cuda()).cpu().numpy().view(np.uint16)

    cores = os.cpu_count() or 1
    yref16, _ = ref.execute(x16, ref.pack(idx, bits), k, n, bits, group, scales, table, workers=cores)
    y64 = orc.reference_f64(x16, idx, bits, group, scales, table)

    y = y16.view(np.float16).astype(np.float64)
    yr = yref16.view(np.float16).astype(np.float64)
    ok_ref, r_ref = _bound_ok(y, yr)
    ok_64, r_64 = _bound_ok(y, y64)
    rep = {"m": m, "k": k, "n": n, "bits": bits, "group": group, "ref_workers": cores,
           "max_ulp_vs_ref": int(_ulp_diff(y16, yref16).max()),
           "rel_l2_vs_ref": float(np.linalg.norm(y - yr) / np.linalg.norm(yr)),
           "max_bound_ratio_vs_ref": r_ref,
           "rel_l2_vs_y64": float(np.linalg.norm(y - y64) / np.linalg.norm(y64)),
           "max_bound_ratio_vs_y64": r_64,
           "ref_rel_l2_vs_y64": float(np.linalg.norm(yr - y64) / np.linalg.norm(y64)),
           "bitwise_equal_to_ref": float(np.mean(y16 == yref16))}
    path = os.environ.get("FLUTE_PARITY_REPORT")
    if path:
        with open(path, "a") as f:
            f.write(json.dumps(rep) + "\n")
    assert ok_ref, f"vs reference engine: {r_ref:.2f}x the bound ({rep})"
    assert ok_64, f"vs binary64: {r_64:.2f}x the bound ({rep})"
