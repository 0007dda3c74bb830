"""GPU parity: the product CUDA path (through the C ABI) vs the CPU oracle.

Bars (BASELINE.json north_star):
  * dequantized LUT values: bit-exact vs vec_dequantize (vec_lut.cpp:39-48),
    exhaustively over every pair and every finite binary16 scale;
  * GEMM: |y - y64| <= 1e-2 * max(|y64|, rms(y64)) per element, y64 = binary64
    product over the f16-rounded dequantized weights; and the
    same bound against the reference engine's own output y_ref;
  * determinism and the reference's bitwise contracts (test_engine.cpp:162-206).
"""
import numpy as np
import pytest

from conftest import f16_bits

pytestmark = pytest.mark.gpu

TOL = 1e-2  # relative, fp16 output (north_star)


def _case(F, orc, rng, m, k, n, bits, group, x_scale=0.5):
    w = rng.standard_normal((k, n)).astype(np.float32)
    idx, scales = F.quantize_matrix(w, bits, group)
    table = F.build_nf_table(bits)
    x16 = f16_bits(orc, rng.standard_normal((m, k)) * x_scale)
    return idx, scales, table, x16


def _within(y16, y64, tol=TOL):
    y = y16.view(np.float16).astype(np.float64)
    bound = tol * np.maximum(np.abs(y64), np.sqrt(np.mean(y64 ** 2)) + 1e-30)
    err = np.abs(y - y64)
    return bool(np.all(err <= bound)), float(err.max()), float((err / bound).max())


def _gemm(F, gpu, idx, scales, table, x16, bits, group, workers=0):
    dw = F.DeviceWeights(idx, scales, table, bits, group)
    x = gpu.from_numpy(x16.view(np.float16)).cuda()
    y = dw.gemm(x, workers=workers)
    gpu.cuda.synchronize()
    return y.cpu().numpy().view(np.uint16), dw


@pytest.mark.parametrize("bits", [2, 3, 4])
def test_dequant_bit_exact_all_pairs_all_scales(F, orc, gpu, bits):
    """Every device-dequantized half2 == vec_dequantize, for all 2^(2b) pairs
    and all 63488 finite binary16 scales (incl. subnormals and negatives)."""
    table = F.build_nf_table(bits)
    vlut = F.make_vectorized_lut(table, bits)
    allh = np.arange(65536, dtype=np.uint32).astype(np.uint16)
    finite = allh[(allh & 0x7C00) != 0x7C00]
    dev = F.dequant_all_device(vlut, bits, finite)
    want = orc.dequant_table(vlut, bits, finite)
    mism = np.count_nonzero(dev != want)
    assert mism == 0, f"{mism} mismatching half2 lookups"


def test_dequant_arbitrary_table(F, orc, gpu):
    """Any LUT (not just NF) — random f16 table values incl. subnormals."""
    rng = np.random.default_rng(5)
    for bits in (2, 3, 4):
        vals = np.sort(rng.standard_normal(1 << bits).astype(np.float32) * 3)
        vals[0] = 3e-6  # subnormal in f16
        vlut = F.make_vectorized_lut(vals, bits)
        sc = f16_bits(orc, rng.uniform(-8, 8, 4096))
        assert np.array_equal(F.dequant_all_device(vlut, bits, sc), orc.dequant_table(vlut, bits, sc))


SMALL = [  # (m, k, n, bits, group)
    (1, 256, 128, 4, 128), (5, 512, 256, 4, 32), (16, 256, 192, 4, 64), (32, 512, 128, 4, 256),
    (1, 512, 256, 3, 128), (7, 256, 128, 3, 32), (32, 384, 320, 3, 64),
    (1, 256, 128, 2, 128), (12, 512, 64, 2, 256), (3, 128, 64, 2, 32),
    (1, 64, 16, 4, 32), (2, 48 * 8, 80, 4, 128), (33, 256, 128, 4, 128), (70, 256, 192, 3, 128),
    # W3 with 9..16 rows: two units per stage (BM = 16); <= 8 rows: four
    (16, 512, 192, 3, 32), (10, 1152, 320, 3, 128), (13, 384, 64, 3, 64),
    (1, 1152, 192, 3, 32), (8, 896, 320, 3, 128), (3, 640, 64, 3, 64),
]


@pytest.mark.parametrize("m,k,n,bits,group", SMALL)
def test_qgemm_vs_oracle_small(F, orc, gpu, m, k, n, bits, group):
    rng = np.random.default_rng(1000 + m * 7 + k + n + bits * 3 + group)
    idx, scales, table, x16 = _case(F, orc, rng, m, k, n, bits, group)
    y16, _ = _gemm(F, gpu, idx, scales, table, x16, bits, group)
    y64 = orc.reference_f64(x16, idx, bits, group, scales, table)
    ok, err, ratio = _within(y16, y64)
    assert ok, f"max err {err:.4g} ({ratio:.2f}x bound)"


@pytest.mark.parametrize("workers", [1, 2, 3, 7, 16, 148, 300])
def test_qgemm_workers_sweep_vs_reference_engine(F, orc, gpu, workers):
    """Stream-K with P CTAs (incl. P > SM count -> ticketed worker ids) vs the
    reference engine's own output at the reference layout (y_ref) and y64."""
    rng = np.random.default_rng(workers)
    m, k, n, bits, group = 9, 1024, 512, 4, 128
    idx, scales, table, x16 = _case(F, orc, rng, m, k, n, bits, group)
    y16, _ = _gemm(F, gpu, idx, scales, table, x16, bits, group, workers=workers)
    y64 = orc.reference_f64(x16, idx, bits, group, scales, table)
    assert _within(y16, y64)[0]
    slices = orc.pack(idx, bits)
    yref, _ = orc.execute(x16, slices, k, n, bits, group, scales, table, workers=min(workers, 8))
    ok, err, _ = _within(y16, yref.view(np.float16).astype(np.float64))
    assert ok, err


@pytest.mark.parametrize("m", [14, 5])
@pytest.mark.parametrize("workers", [1, 5, 37, 148, 300])
def test_qgemm_w3_workers_sweep(F, orc, gpu, workers, m):
    """W3 with multi-unit stages (M <= 8: four units, 9..16: two): odd
    Stream-K ranges split a stage; same bound, bitwise reproducible."""
    rng = np.random.default_rng(300 + workers + m)
    k, n, bits, group = 1664, 320, 3, 128   # 13 k-units: odd per tile
    idx, scales, table, x16 = _case(F, orc, rng, m, k, n, bits, group)
    y16, dw = _gemm(F, gpu, idx, scales, table, x16, bits, group, workers=workers)
    y64 = orc.reference_f64(x16, idx, bits, group, scales, table)
    ok, err, ratio = _within(y16, y64)
    assert ok, f"max err {err:.4g} ({ratio:.2f}x bound)"
    x = gpu.from_numpy(x16.view(np.float16)).cuda()
    assert np.array_equal(dw.gemm(x, workers=workers).cpu().numpy().view(np.uint16), y16)


def test_qgemm_deterministic_and_split_free_bitwise(F, orc, gpu):
    """Bitwise reproducible across runs; P=1 == P=2 when no tile is split
    (test_engine.cpp:183-206 restated for the device unit grid)."""
    rng = np.random.default_rng(7)
    m, k, n, bits, group = 4, 512, 256, 3, 64   # device grid: 4 n-tiles x 4 k-tiles
    idx, scales, table, x16 = _case(F, orc, rng, m, k, n, bits, group)
    dw = F.DeviceWeights(idx, scales, table, bits, group)
    x = gpu.from_numpy(x16.view(np.float16)).cuda()
    outs = [dw.gemm(x, workers=P).cpu().numpy().view(np.uint16) for P in (1, 1, 2, 4)]
    assert np.array_equal(outs[0], outs[1])
    assert np.array_equal(outs[0], outs[2]) and np.array_equal(outs[0], outs[3])
    splits = [dw.gemm(x, workers=P).cpu().numpy().view(np.uint16) for P in (3, 3)]
    assert np.array_equal(splits[0], splits[1])


def test_host_e2e_equals_device_path(F, orc, gpu):
    rng = np.random.default_rng(11)
    m, k, n, bits, group = 3, 1024, 384, 4, 128
    idx, scales, table, x16 = _case(F, orc, rng, m, k, n, bits, group)
    y_dev, dw = _gemm(F, gpu, idx, scales, table, x16, bits, group)
    assert np.array_equal(dw.gemm_host(x16), y_dev)


def test_device_layout_upload_path(F, orc, gpu):
    """flute_weights_create from device-layout buffers == from indices."""
    rng = np.random.default_rng(12)
    m, k, n, bits, group = 2, 512, 128, 3, 128
    idx, scales, table, x16 = _case(F, orc, rng, m, k, n, bits, group)
    y_a, _ = _gemm(F, gpu, idx, scales, table, x16, bits, group)
    dw = F.DeviceWeights.from_device_layout(F.pack_device(idx, bits, group),
                                            F.scales_device(scales, k, n, group),
                                            F.make_vectorized_lut(table, bits), k, n, bits, group)
    assert np.array_equal(dw.gemm_host(x16), y_a)


def test_raw_qgemm_abi(F, orc, gpu):
    """flute_qgemm with caller-owned device buffers and workspace."""
    torch = gpu
    rng = np.random.default_rng(13)
    m, k, n, bits, group = 8, 768, 320, 2, 64
    idx, scales, table, x16 = _case(F, orc, rng, m, k, n, bits, group)
    wdev = torch.from_numpy(F.pack_device(idx, bits, group)).cuda()
    sdev = torch.from_numpy(F.scales_device(scales, k, n, group).view(np.int16)).cuda()
    vdev = torch.from_numpy(F.vlut_device_words(F.make_vectorized_lut(table, bits), bits)
                            .view(np.int32)).cuda()
    ws = torch.zeros(F.workspace_bytes(m, 148), dtype=torch.uint8, device="cuda")
    x = torch.from_numpy(x16.view(np.float16)).cuda()
    y = F.qgemm(x, wdev, sdev, vdev, bits, group, n, ws, workers=0)
    torch.cuda.synchronize()
    y64 = orc.reference_f64(x16, idx, bits, group, scales, table)
    assert _within(y.cpu().numpy().view(np.uint16), y64)[0]
    # the workspace is left zeroed (flags re-armed) -> a second call is identical
    y2 = F.qgemm(x, wdev, sdev, vdev, bits, group, n, ws, workers=0)
    assert torch.equal(y, y2)
    P = F.default_workers(m, k, n, bits)
    assert int(ws[: 4 * (P + 2)].sum()) == 0   # flags + ticket counters back to zero


def test_reference_engine_cases(F, orc, gpu):
    """test_engine.cpp:81-139 restated: constant column, identity activations."""
    # identity X reproduces dequantized rows to one f16 rounding
    rng = np.random.default_rng(0xE1)
    k, n, bits, group = 32, 16, 4, 32
    w = rng.standard_normal((k, n)).astype(np.float32)
    idx, scales = F.quantize_matrix(w, bits, group)
    table = F.build_nf_table(bits)
    x16 = f16_bits(orc, np.eye(k))
    y16, _ = _gemm(F, gpu, idx, scales, table, x16, bits, group)
    deq = np.array([[orc.f16_to_f32(
        orc.vec_dequantize(F.make_vectorized_lut(table, bits)[int(idx[i, j]) << bits],
                           int(scales[j * (k // group) + i // group])) & 0xFFFF)
        for j in range(n)] for i in range(k)])
    assert np.array_equal(y16.view(np.float16).astype(np.float64), deq)


@pytest.mark.parametrize("case", ["identity", "zero", "random", "deterministic", "odd_dims"])
def test_mma_fragment_tensor_core(F, orc, gpu, case):
    """test_mma.cpp:26-100 restated against the tensor-core mma_fragment."""
    rng = np.random.default_rng(0xACC)
    if case == "identity":
        a = f16_bits(orc, np.eye(4)); b = f16_bits(orc, rng.uniform(-4, 4, (4, 3)))
        c = F.mma_fragment(a, b, np.zeros((4, 3)))
        assert np.array_equal(c, b.view(np.float16).astype(np.float32))
    elif case == "zero":
        a = np.zeros((2, 2), np.uint16); b = f16_bits(orc, rng.uniform(-1, 1, (2, 2)))
        c0 = np.array([[1.5, -2.25], [0.125, 3.0]], np.float32)
        assert np.array_equal(F.mma_fragment(a, b, c0), c0)
    elif case in ("random", "deterministic"):
        for _ in range(50 if case == "random" else 1):
            a = f16_bits(orc, rng.uniform(-1, 1, (16, 16))); b = f16_bits(orc, rng.uniform(-1, 1, (16, 8)))
            c = F.mma_fragment(a, b, np.zeros((16, 8)))
            af = a.view(np.float16).astype(np.float64); bf = b.view(np.float16).astype(np.float64)
            ref = af @ bf
            bound = 16 * 2.0 ** -24 * np.abs(af).max(1)[:, None] * np.abs(bf).max(0)[None, :]
            assert np.all(np.abs(c - ref) <= bound)
            if case == "deterministic":
                assert np.array_equal(c, F.mma_fragment(a, b, np.zeros((16, 8))))
    else:
        a = f16_bits(orc, rng.uniform(-1, 1, (5, 7))); b = f16_bits(orc, rng.uniform(-1, 1, (7, 3)))
        c = F.mma_fragment(a, b, np.ones((5, 3)))
        ref = 1 + a.view(np.float16).astype(np.float64) @ b.view(np.float16).astype(np.float64)
        assert np.allclose(c, ref, atol=1e-5)


def test_gpu_error_paths(F, orc, gpu):
    rng = np.random.default_rng(1)
    idx = rng.integers(0, 16, (64, 48)).astype(np.uint8)
    table = F.build_nf_table(4)
    with pytest.raises(F.ConfigError):   # n not a multiple of 16
        F.DeviceWeights(idx[:, :40], np.ones(40 * 2, np.uint16), table, 4, 32)
    with pytest.raises(F.ConfigError):   # group does not divide k
        F.DeviceWeights(idx, np.ones(48, np.uint16), table, 4, 128)
    with pytest.raises(F.InputError):    # index >= 2^bits
        F.DeviceWeights(idx, np.ones(48 * 2, np.uint16), F.build_nf_table(3), 3, 32)
    dw = F.DeviceWeights(idx, np.ones(48 * 2, np.uint16), table, 4, 32)
    with pytest.raises(F.InputError):
        dw.gemm(gpu.zeros((2, 32), dtype=gpu.float16, device="cuda"))


BASE = [  # BASELINE.json configs at full size (parity by the same bound)
    (1, 4096, 4096, 4, 128), (16, 4096, 4096, 4, 128),
    (1, 4096, 14336, 3, 128), (32, 4096, 14336, 3, 128), (4, 14336, 4096, 3, 128),
    (16, 4096, 14336, 3, 128), (16, 14336, 4096, 3, 128),
    (1, 8192, 8192, 2, 256), (8, 8192, 8192, 4, 32),
    (1, 8192, 28672, 4, 128),                        # configs[3] layer (1 GPU)
    (128, 4096, 4096, 4, 128), (512, 2048, 4096, 4, 128),  # configs[4] (tcgen05 path)
]


@pytest.mark.parametrize("m,k,n,bits,group", BASE)
def test_qgemm_baseline_shapes(F, orc, gpu, m, k, n, bits, group):
    rng = np.random.default_rng(k + n + m + bits)
    idx, scales, table, x16 = _case(F, orc, rng, m, k, n, bits, group)
    y16, dw = _gemm(F, gpu, idx, scales, table, x16, bits, group)
    y64 = orc.reference_f64(x16, idx, bits, group, scales, table)
    ok, err, ratio = _within(y16, y64)
    assert ok, f"max err {err:.4g} ({ratio:.2f}x bound)"
    # size-independent property: linearity in X (y(2x) == 2 y(x) exactly in f16 range)
    x = gpu.from_numpy(x16.view(np.float16)).cuda()
    y2 = dw.gemm(x * 2).cpu().numpy().astype(np.float64)
    y1 = y16.view(np.float16).astype(np.float64)
    normal = np.abs(y1) >= 2.0 ** -14   # f16 subnormal outputs round on a fixed grid
    assert np.array_equal(y2[normal], 2 * y1[normal])


@pytest.mark.parametrize("m,k,n,bits,group,cluster", [
    (1, 512, 256, 4, 128, 2), (5, 1024, 128, 3, 64, 4), (16, 1024, 192, 4, 32, 8),
    (32, 768, 128, 2, 256, 2), (3, 256, 64, 3, 128, 2), (9, 2048, 64, 4, 128, 1),
    (12, 1024, 128, 3, 64, 4), (16, 2048, 64, 3, 32, 8), (2, 1536, 128, 3, 128, 4),
    (7, 2048, 64, 3, 32, 8), (32, 2048, 192, 3, 32, 8), (24, 1024, 128, 2, 64, 4),
    (20, 1024, 64, 4, 128, 2)])
def test_qgemm_cluster_splitk(F, orc, gpu, monkeypatch, m, k, n, bits, group, cluster):
    """Cluster split-K mode (one cluster per 64-column tile, DSMEM reduction),
    forced on small shapes; same bound as the Stream-K path, and bitwise
    reproducible run to run."""
    monkeypatch.setenv("FLUTE_FORCE_CLUSTER", str(cluster))
    rng = np.random.default_rng(77 + m + k + n + bits + cluster)
    idx, scales, table, x16 = _case(F, orc, rng, m, k, n, bits, group)
    y16, dw = _gemm(F, gpu, idx, scales, table, x16, bits, group)
    y64 = orc.reference_f64(x16, idx, bits, group, scales, table)
    ok, emax, ratio = _within(y16, y64)
    assert ok, f"max err {emax:.4g} ({ratio:.2f} of bound)"
    x = gpu.from_numpy(x16.view(np.float16)).cuda()
    again = dw.gemm(x).cpu().numpy().view(np.uint16)
    assert np.array_equal(again, y16)


TC_CASES = [  # (m, k, n, bits, group, splits) — compute-bound tcgen05 path (m >= 64)
    (64, 256, 128, 4, 128, 1), (64, 1024, 256, 4, 32, 4), (100, 512, 192, 3, 64, 2),
    (128, 512, 384, 2, 256, 1), (200, 384, 320, 4, 128, 3), (256, 1024, 128, 3, 128, 0),
    (512, 2048, 512, 4, 128, 0), (65, 128, 64, 2, 32, 1),
]
# UMMA N = 256 with 64-deep stages (chosen when 128-row tiles need more than one
# wave; forced here): W2/W3/W4, a partial second row block, an odd 64-column
# tile count, group 32 and split K
TC256_CASES = [(300, 512, 192, 3, 32, 0), (256, 384, 320, 2, 64, 3), (512, 1024, 256, 4, 256, 2),
               (257, 256, 64, 4, 128, 1), (512, 2048, 1024, 4, 128, 0)]


@pytest.mark.parametrize("m,k,n,bits,group,splits", TC256_CASES)
def test_qgemm_tcgen05_n256_vs_oracle(F, orc, gpu, monkeypatch, m, k, n, bits, group, splits):
    monkeypatch.setenv("FLUTE_TC_BN", "256")
    if splits:
        monkeypatch.setenv("FLUTE_TC_SPLITS", str(splits))
    rng = np.random.default_rng(7000 + m + k + n + bits + group)
    idx, scales, table, x16 = _case(F, orc, rng, m, k, n, bits, group)
    y16, dw = _gemm(F, gpu, idx, scales, table, x16, bits, group)
    y64 = orc.reference_f64(x16, idx, bits, group, scales, table)
    ok, emax, ratio = _within(y16, y64)
    assert ok, f"max err {emax:.4g} ({ratio:.2f} of bound)"


@pytest.mark.parametrize("m,k,n,bits,group,splits", TC_CASES)
def test_qgemm_tcgen05_vs_oracle(F, orc, gpu, monkeypatch, m, k, n, bits, group, splits):
    """M >= 64 runs the tcgen05/TMEM kernel (UMMA from the dequantised W^T tile
    in swizzled smem, fp32 accumulator in TMEM, optional split-K): same bound
    as the memory-bound path, deterministic run to run."""
    if splits:
        monkeypatch.setenv("FLUTE_TC_SPLITS", str(splits))
    rng = np.random.default_rng(5000 + m + k + n + bits + group)
    idx, scales, table, x16 = _case(F, orc, rng, m, k, n, bits, group)
    y16, dw = _gemm(F, gpu, idx, scales, table, x16, bits, group)
    y64 = orc.reference_f64(x16, idx, bits, group, scales, table)
    ok, emax, ratio = _within(y16, y64)
    assert ok, f"max err {emax:.4g} ({ratio:.2f} of bound)"
    x = gpu.from_numpy(x16.view(np.float16)).cuda()
    assert np.array_equal(dw.gemm(x).cpu().numpy().view(np.uint16), y16)


# Several MMA issuer warps with their own TMEM accumulators (BN = 32 / 64:
# four, BN = 128: two), the 8-slot A ring and the separately released X ring:
# fewer stages than accumulators (k = 128: two 64-k stages), ragged m blocks,
# split K, every bit width, and the M = 16 / 32 regime forced onto tcgen05.
@pytest.mark.parametrize("m,k,n,bits,group,bn,splits", [
    (64, 128, 128, 4, 128, 32, 1), (40, 256, 192, 3, 32, 32, 1), (96, 1024, 256, 2, 64, 32, 2),
    (64, 1024, 320, 4, 128, 64, 0), (100, 512, 128, 3, 128, 64, 3), (128, 2048, 256, 4, 256, 128, 2),
    (130, 384, 192, 2, 128, 128, 1), (16, 1024, 256, 3, 128, 32, 0), (32, 2048, 512, 4, 128, 32, 0),
    (24, 640, 128, 3, 64, 64, 1)])
def test_qgemm_tcgen05_multi_issuer_vs_oracle(F, orc, gpu, monkeypatch, m, k, n, bits, group, bn, splits):
    monkeypatch.setenv("FLUTE_TC_BN", str(bn))
    monkeypatch.setenv("FLUTE_TC_MIN_M", "16")
    if splits:
        monkeypatch.setenv("FLUTE_TC_SPLITS", str(splits))
    rng = np.random.default_rng(9100 + m + k + n + bits + group + bn)
    idx, scales, table, x16 = _case(F, orc, rng, m, k, n, bits, group)
    y16, dw = _gemm(F, gpu, idx, scales, table, x16, bits, group)
    y64 = orc.reference_f64(x16, idx, bits, group, scales, table)
    ok, emax, ratio = _within(y16, y64)
    assert ok, f"max err {emax:.4g} ({ratio:.2f} of bound)"
    x = gpu.from_numpy(x16.view(np.float16)).cuda()
    for _ in range(2):  # fixed accumulator order: bitwise reproducible
        assert np.array_equal(dw.gemm(x).cpu().numpy().view(np.uint16), y16)


def test_qgemm_tcgen05_matches_mma_path(F, orc, gpu, monkeypatch):
    """The tcgen05 path and the mma.sync path (forced with FLUTE_NO_TC) agree
    within the parity bound on a BASELINE configs[4]-style shape."""
    rng = np.random.default_rng(44)
    m, k, n, bits, group = 256, 4096, 1024, 4, 128
    idx, scales, table, x16 = _case(F, orc, rng, m, k, n, bits, group)
    y_tc, dw = _gemm(F, gpu, idx, scales, table, x16, bits, group)
    monkeypatch.setenv("FLUTE_NO_TC", "1")
    x = gpu.from_numpy(x16.view(np.float16)).cuda()
    y_mma = dw.gemm(x).cpu().numpy().view(np.uint16)
    y64 = orc.reference_f64(x16, idx, bits, group, scales, table)
    assert _within(y_tc, y64)[0] and _within(y_mma, y64)[0]


def test_execute_abi_reference_formats(F, orc, gpu):
    """flute_execute: the reference call (engine.hpp:72) on host buffers in the
    reference's own formats (canonical slices, dup-2 vLUT) — y within the
    bound of the reference engine's output, stats == plan_traffic."""
    rng = np.random.default_rng(31)
    m, k, n, bits, group = 5, 512, 256, 3, 128
    idx, scales, table, x16 = _case(F, orc, rng, m, k, n, bits, group)
    slices = F.reorder_and_split(idx, bits)
    vlut = F.make_vectorized_lut(table, bits, dup=2)
    res = F.execute(x16, slices, k, n, bits, group, scales, vlut, dup=2, workers=3)
    yref, _ = orc.execute(x16, orc.pack(idx, bits), k, n, bits, group, scales, table, workers=3)
    ok, err, _ = _within(res.y, yref.view(np.float16).astype(np.float64))
    assert ok, err
    assert res.stats == F.plan_traffic(m, k, n, bits, group, workers=3)


def test_cuda_graph_capture_without_warmup(F, orc, gpu):
    """A fresh DeviceWeights is capture-safe for every m <= 32 (the workspace
    is sized up front), and for larger m after reserve(); replaying the graph
    reproduces the eager result bit for bit."""
    rng = np.random.default_rng(12)
    k, n, bits, group = 1024, 512, 3, 128
    idx, sc = F.quantize_matrix(rng.standard_normal((k, n)).astype(np.float32), bits, group)
    table = F.build_nf_table(bits)
    st = gpu.cuda.Stream()
    for m in (1, 4, 16, 32, 128):
        dw = F.DeviceWeights(idx, sc, table, bits, group)
        if m > 32:
            dw.reserve(m)
        x = gpu.randn(m, k, dtype=gpu.float16, device="cuda")
        y = gpu.empty(m, n, dtype=gpu.float16, device="cuda")
        g = gpu.cuda.CUDAGraph()
        with gpu.cuda.graph(g, stream=st):
            dw.gemm(x, y, stream=st.cuda_stream)
        g.replay()
        st.synchronize()
        assert np.array_equal(y.cpu().numpy().view(np.uint16), dw.gemm(x).cpu().numpy().view(np.uint16))


def test_autotune_keeps_results_in_bound(F, orc, gpu):
    """autotune() times the candidate decompositions and keeps the fastest;
    later default calls stay within the bound and bitwise reproducible."""
    rng = np.random.default_rng(8)
    m, k, n, bits, group = 4, 2048, 1024, 3, 128
    idx, scales, table, x16 = _case(F, orc, rng, m, k, n, bits, group)
    dw = F.DeviceWeights(idx, scales, table, bits, group)
    report = dw.autotune(m)
    assert report.count("us") >= 2, report
    x = gpu.from_numpy(x16.view(np.float16)).cuda()
    y1 = dw.gemm(x).cpu().numpy().view(np.uint16)
    y2 = dw.gemm(x).cpu().numpy().view(np.uint16)
    assert np.array_equal(y1, y2)
    assert _within(y1, orc.reference_f64(x16, idx, bits, group, scales, table))[0]
    with pytest.raises(F.ConfigError):
        dw.autotune(64)


def test_gemm_host_batch_matches_device_path(F, gpu):
    """flute_gemm_host_batch (pipelined host-buffer batch, bench.py's e2e path)
    returns, item for item, the bits of the device-resident gemm(); a handle
    may repeat inside one batch."""
    torch = gpu
    rng = np.random.default_rng(42)
    shapes = [(256, 320, 3), (512, 128, 4), (384, 192, 2)]
    hs = []
    for (k, n, bits) in shapes:
        idx, sc = F.quantize_matrix(rng.standard_normal((k, n)).astype(np.float32), bits, 128)
        hs.append(F.DeviceWeights(idx, sc, F.build_nf_table(bits), bits, 128))
    items, want = [], []
    for i, m in enumerate([1, 5, 32, 17, 3, 64]):
        dw = hs[i % len(hs)]
        x = (rng.standard_normal((m, dw.k)) * 0.5).astype(np.float16)
        xd = torch.from_numpy(x).cuda()
        want.append(dw.gemm(xd).cpu().numpy().view(np.uint16))
        items.append((dw, x.view(np.uint16), np.zeros((m, dw.n), np.uint16)))
    F.gemm_host_batch(items)
    for (_, _, out), w in zip(items, want):
        assert np.array_equal(out, w)
    with pytest.raises(F.InputError):
        F.gemm_host_batch([(hs[0], np.zeros((2, hs[0].k + 1), np.uint16), np.zeros((2, hs[0].n), np.uint16))])


def test_mixed_m_on_one_handle_keeps_streamk_workspace_clean(F, gpu):
    """Regression: the tcgen05 path's split-K partials share the handle's
    workspace with the Stream-K fixup slots (zero = unwritten); a prefill-sized
    call (M >= 64) between decode-sized calls must not perturb them."""
    torch = gpu
    rng = np.random.default_rng(5)
    k, n = 384, 192
    idx, sc = F.quantize_matrix(rng.standard_normal((k, n)).astype(np.float32), 2, 128)
    dw = F.DeviceWeights(idx, sc, F.build_nf_table(2), 2, 128)
    x32 = torch.from_numpy((rng.standard_normal((32, k)) * 0.5).astype(np.float16)).cuda()
    x64 = torch.from_numpy((rng.standard_normal((64, k)) * 0.5).astype(np.float16)).cuda()
    first = dw.gemm(x32).cpu().numpy().view(np.uint16)
    big = dw.gemm(x64).cpu().numpy().view(np.uint16)
    for _ in range(4):
        assert np.array_equal(dw.gemm(x64).cpu().numpy().view(np.uint16), big)
        assert np.array_equal(dw.gemm(x32).cpu().numpy().view(np.uint16), first)


@pytest.mark.parametrize("graph", [True, False])
def test_host_batch_object_replays(F, gpu, graph):
    """HostBatch (CUDA-graph capture of copies + GEMMs + copies, or the eager
    pipelined path) gives the device path's bits, including an M >= 64
    (tcgen05) item, and picks up refilled inputs on every run."""
    torch = gpu
    rng = np.random.default_rng(7)
    hs = []
    for (k, n, bits) in [(256, 320, 3), (512, 256, 4)]:
        idx, sc = F.quantize_matrix(rng.standard_normal((k, n)).astype(np.float32), bits, 128)
        hs.append(F.DeviceWeights(idx, sc, F.build_nf_table(bits), bits, 128))
    ms = [1, 16, 64, 32]
    xs = [np.zeros((m, hs[i % 2].k), np.uint16) for i, m in enumerate(ms)]
    outs = [np.zeros((m, hs[i % 2].n), np.uint16) for i, m in enumerate(ms)]
    batch = F.HostBatch([(hs[i % 2], xs[i], outs[i]) for i in range(len(ms))], graph=graph)
    for rep in range(3):
        want = []
        for i, m in enumerate(ms):
            x = (rng.standard_normal((m, hs[i % 2].k)) * 0.5).astype(np.float16)
            xs[i][...] = x.view(np.uint16)
            want.append(hs[i % 2].gemm(torch.from_numpy(x).cuda()).cpu().numpy().view(np.uint16))
        batch.run()
        for o, w in zip(outs, want):
            assert np.array_equal(o, w), rep


def _random_w3_cases(count=32, seed=2024):
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(count):
        m = int(rng.integers(1, 33))
        k = 128 * int(rng.integers(1, 24))
        n = 64 * int(rng.integers(1, 12)) - (16 if rng.random() < 0.3 else 0)
        group = int(rng.choice([32, 64, 128, 256]))
        while k % group:
            group //= 2
        workers = int(rng.choice([0, 0, 1, 3, 29, 148, 296]))
        out.append((m, k, n, group, workers))
    return out


@pytest.mark.parametrize("m,k,n,group,workers", _random_w3_cases())
def test_qgemm_w3_random_shapes(F, orc, gpu, m, k, n, group, workers):
    """Randomised W3 shapes through the M <= 32 kernels (multi-unit stages for
    M <= 16, two 4-warp CTAs per SM for 17..32): ragged k-unit counts, partial
    64-column tiles, every group size, default and explicit Stream-K worker
    counts."""
    rng = np.random.default_rng(m * 1000003 + k * 101 + n + group + workers)
    idx, scales, table, x16 = _case(F, orc, rng, m, k, n, 3, group)
    y16, _ = _gemm(F, gpu, idx, scales, table, x16, 3, group, workers=workers)
    y64 = orc.reference_f64(x16, idx, 3, group, scales, table)
    ok, err, ratio = _within(y16, y64)
    assert ok, f"max err {err:.4g} ({ratio:.2f}x bound)"
