"""GPU weight preparation: the device quantizer is
bit-exact with quantize_matrix (itself pinned to the reference library), the
on-device packer reproduces the host device layout, and an FLTE container
written by the reference uploads (canonical slices re-permuted on the GPU) to
weights that give the same GEMM bits as the host-packed path."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "flte.npz")


@pytest.mark.parametrize("bits,group,k,n", [(2, 32, 256, 96), (3, 128, 512, 256), (4, 64, 384, 200),
                                            (4, 256, 1024, 64), (3, 32, 128, 1000)])
def test_quantize_device_bit_exact(F, gpu, bits, group, k, n):
    rng = np.random.default_rng(bits * 1000 + group + n)
    w = (rng.standard_normal((k, n)) * rng.uniform(1e-3, 30, (1, n))).astype(np.float32)
    w[:group, 3 % n] = 0.0            # a zero group
    w[group:2 * group, 5 % n] = -1.0  # constant group
    idx_h, sc_h = F.quantize_matrix(w, bits, group)
    idx_d, sc_d = F.quantize_matrix_device(gpu.from_numpy(w).cuda(), bits, group)
    assert np.array_equal(idx_d.cpu().numpy(), idx_h)
    assert np.array_equal(sc_d.cpu().numpy().view(np.uint16), sc_h)


def test_quantize_device_rejects_nonfinite(F, gpu):
    w = np.ones((128, 64), np.float32)
    w[5, 7] = np.inf
    with pytest.raises(F.InputError):
        F.quantize_matrix_device(gpu.from_numpy(w).cuda(), 4, 128)


@pytest.mark.parametrize("bits", [2, 3, 4])
def test_device_packing_matches_host_gemm_bits(F, orc, gpu, bits):
    """Weights built on the device (quantize -> pack, all on the GPU) give the
    same GEMM bits as the host-packed DeviceWeights."""
    rng = np.random.default_rng(bits)
    k, n, group, m = 512, 320, 128, 3
    w = rng.standard_normal((k, n)).astype(np.float32)
    idx_d, sc_d = F.quantize_matrix_device(gpu.from_numpy(w).cuda(), bits, group)
    table = F.build_nf_table(bits)
    t16 = table.astype(np.float16).view(np.uint16)
    dw_dev = F.DeviceWeights.from_device_indices(idx_d, sc_d, t16, bits, group)
    dw_host = F.DeviceWeights(idx_d.cpu().numpy(), sc_d.cpu().numpy().view(np.uint16), table, bits,
                              group)
    x = gpu.randn(m, k, dtype=gpu.float16, device="cuda")
    assert np.array_equal(dw_dev.gemm(x).cpu().numpy().view(np.uint16),
                          dw_host.gemm(x).cpu().numpy().view(np.uint16))


def test_flte_upload_matches_host_path(F, orc, gpu):
    """Reference-written FLTE containers -> DeviceWeights.from_flte: same GEMM
    bits as uploading the same indices through the host packer."""
    gold = np.load(GOLD)
    for i, (bits, group, k, n) in enumerate(gold["meta"]):
        bits, group, k, n = int(bits), int(group), int(k), int(n)
        blob = gold[f"flte{i}"].tobytes()
        dw_f = F.DeviceWeights.from_flte(blob)
        idx, sc = F.quantize_matrix(gold[f"w{i}"], bits, group)
        dw_h = F.DeviceWeights(idx, sc, F.build_nf_table(bits), bits, group)
        x = gpu.randn(5, k, dtype=gpu.float16, device="cuda")
        assert np.array_equal(dw_f.gemm(x).cpu().numpy().view(np.uint16),
                              dw_h.gemm(x).cpu().numpy().view(np.uint16))
