"""Learned-sigma refinement (reference quantize.cpp:
141-282).

CPU: the plain-C restatement (oracle/flute_oracle.c orc_ste_evaluate /
orc_refine_scales) is pinned BIT-FOR-BIT to the reference library (loss,
gradients, indices, sigma trajectory, folded scales, failing step).
GPU: the product (csrc/refine_kernels.cu through the C ABI) against that
oracle — indices, gradients, sigma and folded scales bit-identical (explicit
binary64 mul/add in the reference's order), losses within 1e-12 relative
(the loss is a fixed-order tree sum instead of the reference's sequential
sum)."""
import numpy as np
import pytest

LOSS_RTOL = 1e-12

CASES = [  # k, n, m, bits, group
    (64, 8, 8, 4, 32), (256, 24, 16, 3, 64), (128, 16, 4, 2, 128), (512, 40, 33, 4, 256),
    (96, 5, 1, 3, 32),
]


def _inputs(k, n, m, group, seed, zero_group=True):
    rng = np.random.default_rng(seed)
    w = (rng.standard_normal((k, n)) * rng.uniform(0.2, 3.0, (1, n))).astype(np.float32)
    if zero_group and n > 2:
        w[:group, 1] = 0.0
    x = rng.standard_normal((m, k)).astype(np.float32)
    sigma = rng.uniform(0.8, 1.2, k // group * n)
    return w, x, sigma


def _refine(lib, exc, *args):
    try:
        return lib.refine_scales(*args)
    except exc as e:
        return ("failed", e.step)


# --------------------------------------------------------------------- CPU
@pytest.mark.parametrize("k,n,m,bits,group", CASES)
def test_oracle_ste_matches_reference_bitwise(orc, ref, k, n, m, bits, group):
    w, x, s = _inputs(k, n, m, group, k + n + m)
    s = s * orc.nf_sigma()
    lo, go, io = orc.ste_evaluate(w, x, bits, group, s)
    lr, gr, ir = ref.ste_evaluate(w, x, bits, group, s)
    assert lo == lr
    assert np.array_equal(go, gr)
    assert np.array_equal(io, ir)


@pytest.mark.parametrize("k,n,m,bits,group", CASES)
@pytest.mark.parametrize("steps,lr", [(0, 1e-3), (12, 1e-5), (5, 1e40)])
def test_oracle_refine_matches_reference_bitwise(orc, ref, k, n, m, bits, group, steps, lr):
    import oracle
    w, x, _ = _inputs(k, n, m, group, 3 * k + n)
    a = _refine(orc, oracle.RefineFailed, w, x, bits, group, steps, lr)
    b = _refine(ref, oracle.RefineFailed, w, x, bits, group, steps, lr)
    if isinstance(a, tuple) or isinstance(b, tuple):
        assert a == b
        return
    for key in ("indices", "scales", "sigma"):
        assert np.array_equal(a[key], b[key]), key
    assert a["initial_loss"] == b["initial_loss"] and a["final_loss"] == b["final_loss"]


# --------------------------------------------------------------------- GPU
@pytest.mark.gpu
@pytest.mark.parametrize("k,n,m,bits,group", CASES + [(1024, 384, 64, 3, 128)])
def test_ste_evaluate_gpu_matches_oracle(F, orc, gpu, k, n, m, bits, group):
    w, x, s = _inputs(k, n, m, group, 7 * k + n)
    s = s * orc.nf_sigma()
    lg, gg, ig = F.ste_evaluate(w, x, bits, group, s)
    lo, go, io = orc.ste_evaluate(w, x, bits, group, s)
    assert np.array_equal(ig, io)
    assert np.array_equal(gg, go)  # bit-identical gradients
    assert abs(lg - lo) <= LOSS_RTOL * abs(lo)


@pytest.mark.gpu
@pytest.mark.parametrize("k,n,m,bits,group", CASES + [(512, 256, 32, 4, 64)])
@pytest.mark.parametrize("steps,lr", [(0, 1e-3), (12, 1e-5), (30, 2e-5), (5, 1e40)])
def test_refine_scales_gpu_matches_oracle(F, orc, gpu, k, n, m, bits, group, steps, lr):
    import oracle
    w, x, _ = _inputs(k, n, m, group, 5 * k + n)
    a = _refine(F, F.OptimizationError, w, x, bits, group, steps, lr)
    b = _refine(orc, oracle.RefineFailed, w, x, bits, group, steps, lr)
    if isinstance(a, tuple) or isinstance(b, tuple):
        assert a == b
        return
    for key in ("indices", "scales", "sigma"):
        assert np.array_equal(a[key], b[key]), key
    for key in ("initial_loss", "final_loss"):
        assert abs(a[key] - b[key]) <= LOSS_RTOL * abs(b[key]), key


@pytest.mark.gpu
def test_refine_steps0_is_plain_quantization(F, gpu):
    w, x, _ = _inputs(256, 32, 8, 64, 11)
    r = F.refine_scales(w, x, 3, 64, 0, 1e-3)
    idx, sc = F.quantize_matrix(w, 3, 64)
    assert np.array_equal(r["indices"], idx) and np.array_equal(r["scales"], sc)
    assert r["initial_loss"] == r["final_loss"]


@pytest.mark.gpu
def test_refine_errors(F, gpu):
    w, x, s = _inputs(64, 4, 4, 32, 1)
    with pytest.raises(F.InputError):
        F.refine_scales(w, x, 4, 32, -1, 1e-3)
    with pytest.raises(F.InputError):
        F.ste_evaluate(w, x[:, :32], 4, 32, s)  # x columns != w rows
    with pytest.raises(F.InputError):
        F.ste_evaluate(w, x, 4, 32, s[:-1])     # sigma group count
    with pytest.raises(F.ConfigError):
        F.ste_evaluate(w, x, 5, 32, s)
    bad = w.copy()
    bad[40, 2] = np.nan
    bad[3, 3] = np.inf
    with pytest.raises(F.InputError, match=r"\(40, 2\)"):  # first hit in the reference's j-major scan
        F.ste_evaluate(bad, x, 4, 32, s)


@pytest.mark.gpu
def test_refine_descends_at_llm_scale(F, gpu):
    """Size-independent property at a layer-sized problem: a small-rate
    descent lowers the calibration loss and keeps every folded scale finite."""
    rng = np.random.default_rng(0)
    k, n, m = 4096, 1024, 64
    w = (rng.standard_t(3, (k, n)) * 0.02).astype(np.float32)
    x = rng.standard_normal((m, k)).astype(np.float32)
    r = F.refine_scales(w, x, 4, 128, 4, 1e-4)
    assert r["final_loss"] < r["initial_loss"]
    assert np.all((r["scales"] & 0x7C00) != 0x7C00)
