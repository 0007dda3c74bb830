"""Product host layer (C++ behind the C ABI) vs the pinned oracle and the
reference's golden fixtures — CPU only, no kernel launches."""
import os
import re

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(__file__), "golden")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def gold(name):
    return np.load(os.path.join(GOLD, name))


def test_library_exports_every_declared_symbol(F):
    """libflute_b200.so loads and exports every function include/flute_c.h declares."""
    import ctypes
    hdr = open(os.path.join(ROOT, "include", "flute_c.h")).read()
    declared = set(re.findall(r"\b(flute_[a-z0-9_]+)\s*\(", hdr))
    lib = ctypes.CDLL(F.LIB_PATH)
    missing = [s for s in sorted(declared) if not hasattr(lib, s)]
    assert not missing, missing
    assert declared == set(F.exported_symbols())


def test_numerics_and_tables(F):
    g = gold("numerics.npz")
    got = np.array([F.f32_to_f16(v) for v in g["f32"][:3000]], np.uint16)
    assert np.array_equal(got, g["f16"][:3000])
    t = gold("nf_tables.npz")
    for b in (2, 3, 4):
        assert np.array_equal(F.build_nf_table(b), t[f"nf{b}"])


def test_quantize_pack_vlut_golden(F):
    g = gold("quant_pack.npz")
    layouts = [tuple(l) for l in g["layouts"]]
    for bits in (2, 3, 4):
        for group in (32, 64):
            key = f"b{bits}g{group}"
            idx, sc = F.quantize_matrix(g[f"{key}_w"], bits, group)
            assert np.array_equal(idx, g[f"{key}_idx"]) and np.array_equal(sc, g[f"{key}_scales"])
            for li, L in enumerate(layouts):
                sl = F.reorder_and_split(idx, bits, L)
                for si, s in enumerate(sl):
                    assert np.array_equal(s, g[f"{key}_L{li}_s{si}"])
                assert np.array_equal(F.unpack_matrix(sl, *idx.shape, bits, L), idx)
        assert np.array_equal(F.make_vectorized_lut(F.build_nf_table(bits), bits), g[f"vlut{bits}"])


def test_vlut_dup_interleave_and_known_answers(F, orc):  # test_vec_lut.cpp:11-62
    t = F.build_nf_table(4)
    v1 = F.make_vectorized_lut(t, 4, 1)
    v4 = F.make_vectorized_lut(t, 4, 4)
    assert v1.size == 256 and v4.size == 1024
    assert np.array_equal(v4.reshape(256, 4), np.repeat(v1[:, None], 4, axis=1))  # e*d + c
    r = F.vec_dequantize((15 << 4) | 0, F.f32_to_f16(2.0), v1, 4)
    assert F.f16_to_f32(r & 0xFFFF) == 2.0 and F.f16_to_f32(r >> 16) == -2.0
    for bad in (0, 3):
        with pytest.raises(F.ConfigError):
            F.make_vectorized_lut(t, 4, bad)
    with pytest.raises(F.InputError):
        F.vec_dequantize(256, F.f32_to_f16(1.0), v1, 4)


def test_vec_dequantize_matches_oracle(F, orc):
    rng = np.random.default_rng(3)
    for bits in (2, 3, 4):
        v = F.make_vectorized_lut(F.build_nf_table(bits), bits)
        for _ in range(200):
            p = int(rng.integers(0, 1 << (2 * bits)))
            s = int(rng.integers(0, 0x7C00)) | (int(rng.integers(0, 2)) << 15)
            assert F.vec_dequantize(p, s, v, bits) == orc.vec_dequantize(int(v[p]), s)


@pytest.mark.parametrize("bits", [2, 3, 4])
@pytest.mark.parametrize("k,n,group", [(128, 64, 32), (512, 192, 128), (384, 80, 64),
                                         (64, 16, 32), (768, 256, 256)])
def test_device_layout_bijective(F, bits, k, n, group):
    """unpack_device(pack_device(Q)) == Q; canonical -> device repack agrees;
    padded geometry as documented."""
    rng = np.random.default_rng(k * n + bits)
    idx = rng.integers(0, 1 << bits, (k, n)).astype(np.uint8)
    dev = F.pack_device(idx, bits, group)
    kp, np_ = -(-k // 128) * 128, -(-n // 64) * 64
    assert dev.size == kp * np_ * bits // 8
    assert np.array_equal(F.unpack_device(dev, k, n, bits, group), idx)
    if k % 64 == 0 and n % 64 == 0:
        sl = F.reorder_and_split(idx, bits)
        assert np.array_equal(F.repack_canonical(sl, k, n, bits, group), dev)


def test_device_layout_w4_register_order(F):
    """Byte p of lane word j holds pair (n=16j+g+8(p&1), k=2t+8(p>>1)), first in
    the high nibble."""
    k, n = 128, 64
    idx = np.zeros((k, n), np.uint8)
    idx[10, 21] = 0xA   # k=10 -> t=1, p>>1=1 ; n=21 -> j=1, g=5, p&1=0
    idx[11, 21] = 0x3
    dev = F.pack_device(idx, 4, 128)
    lane = 5 * 4 + 1
    # warp 0 (k in 0..15), lane, word j=1, byte p=2
    assert dev[(0 * 32 + lane) * 16 + 1 * 4 + 2] == 0xA3
    assert np.count_nonzero(dev) == 1


def test_device_layout_w3_lane_words(F):
    """W3 lane words: the 6-bit pair index D = (hi_k<<2|hi_k1)<<2
    | (lo_k<<1|lo_k1) of atoms 0/1/2 sits in bits 0..5 of byte p of word A / B
    / C; atom 3's D is spread over bits 6..7 of byte p of A (bits 0-1), B
    (2-3) and C (4-5).  A, B are the lane's 8 bytes in the unit's first 2 KiB,
    C its 4 bytes in the last 1 KiB."""
    k, n = 128, 64
    def one(row, col, a, b):
        idx = np.zeros((k, n), np.uint8)
        idx[row, col], idx[row + 1, col] = a, b
        return F.pack_device(idx, 3, 128)
    # pair (k=10,11) at column 21: t=1, p>>1=1, j=1, g=5, p&1=0 -> byte p=2
    a, b = 6, 5  # hi 3 / 2, lo 0 / 1 -> D = (3<<2|2)<<2 | (0<<1|1) = 57
    dev = one(10, 21, a, b)
    lane = 5 * 4 + 1
    assert dev[lane * 8 + 4 + 2] == 57          # word B (atom 1), byte 2
    assert np.count_nonzero(dev) == 1
    # the same pair at column 53 (atom j=3, g=5): D split over A/B/C bits 6..7
    dev = one(10, 53, a, b)
    assert dev[lane * 8 + 0 + 2] == (57 & 3) << 6          # A byte 2
    assert dev[lane * 8 + 4 + 2] == ((57 >> 2) & 3) << 6   # B byte 2
    assert dev[2048 + lane * 4 + 2] == ((57 >> 4) & 3) << 6  # C byte 2
    assert np.count_nonzero(dev) == 3
    for col in (21, 53):
        d = one(10, col, a, b)
        back = F.unpack_device(d, k, n, 3, 128)
        assert back[10, col] == a and back[11, col] == b


def test_scales_device_layout(F):
    k, n, group = 256, 128, 64
    sc = np.arange(n * (k // group), dtype=np.uint16) + 1
    d = F.scales_device(sc, k, n, group)
    gp = 256 // 64
    # column col, group G -> block (col//64, G), slot (col%8)*8 + (col%64//16)*2 + (col%16)//8
    for col in (0, 7, 8, 15, 16, 63, 64, 127):
        for G in range(gp):
            slot = (col % 8) * 8 + ((col % 64) // 16) * 2 + (col % 16) // 8
            assert d[((col // 64) * gp + G) * 64 + slot] == sc[col * (k // group) + G]


def test_device_vlut_permutation_3bit(F):
    v = F.make_vectorized_lut(F.build_nf_table(3), 3)
    d = F.vlut_device_words(v, 3)
    for ik in range(8):
        for ik1 in range(8):
            dev_index = ((ik >> 1) << 4) | ((ik1 >> 1) << 2) | ((ik & 1) << 1) | (ik1 & 1)
            assert d[dev_index] == v[(ik << 3) | ik1]
    for bits in (2, 4):
        v = F.make_vectorized_lut(F.build_nf_table(bits), bits)
        assert np.array_equal(F.vlut_device_words(v, bits), v)


def test_streamk_plan_golden(F):
    g = gold("streamk.npz")
    for key in {k.rsplit("_", 1)[0] for k in g.files}:
        tm, tn, tk, P = (int(v) for v in key[1:].split("_"))
        p = F.plan_stream_k(tm, tn, tk, P)
        assert np.array_equal(p.ranges, g[key + "_ranges"])
        assert np.array_equal(p.fixups, g[key + "_fixups"])
        assert p.total_slots == int(g[key + "_slots"][0])
    with pytest.raises(F.ConfigError):
        F.plan_stream_k(0, 1, 1, 1)
    with pytest.raises(F.ConfigError):
        F.plan_stream_k(1, 1, 1, 0)


def test_plan_traffic_golden_and_oracle(F, orc):
    g = gold("engine.npz")
    for ci in range(len([k for k in g.files if k.endswith("_meta")])):
        m, k, n, bits, group, P = (int(v) for v in g[f"c{ci}_meta"])
        st = F.plan_traffic(m, k, n, bits, group, workers=P)
        assert list(st.values()) == [int(v) for v in g[f"c{ci}_plan_traffic"]]
        # execute().stats == plan_traffic (reference engine.hpp:83-96 contract)
        assert list(st.values()) == [int(v) for v in g[f"c{ci}_stats"]]
    for P in (1, 3, 8, 148):
        a = F.plan_traffic(4, 1024, 512, 3, 128, workers=P, stages=4, tile_m=32)
        b = orc.plan_traffic(4, 1024, 512, 3, 128, workers=P, stages=4, tile_m=32)
        assert list(a.values()) == [int(v) for v in b]


def test_bits_per_param(F):  # test_engine.cpp:276-283
    assert F.bits_per_param(4, 32) == 4.5 and F.bits_per_param(4, 64) == 4.25
    assert F.bits_per_param(4, 128) == 4.125 and F.bits_per_param(4, 256) == 4.0625
    assert F.bits_per_param(3, 128) == 3.125 and F.bits_per_param(3, 256) == 3.0625
    with pytest.raises(F.ConfigError):
        F.bits_per_param(5, 128)


def test_error_taxonomy(F):
    """ConfigError / InputError mapping mirrors the reference (errors.hpp)."""
    idx = np.zeros((64, 48), np.uint8)
    with pytest.raises(F.ConfigError):
        F.reorder_and_split(idx, 4, (16, 32, 48, 16, 8, 16))
    with pytest.raises(F.ConfigError):
        F.reorder_and_split(idx, 4, (16, 16, 15, 16, 8, 15))
    with pytest.raises(F.ConfigError):
        F.quantize_matrix(np.zeros((100, 16), np.float32), 4, 128)
    with pytest.raises(F.InputError):
        F.quantize_matrix(np.full((32, 16), np.inf, np.float32), 4, 32)
    with pytest.raises(F.ConfigError):
        F.pack_device(np.zeros((64, 40), np.uint8), 4, 32)   # n % 16
    with pytest.raises(F.InputError):
        F.pack_device(np.full((64, 48), 9, np.uint8), 3, 32)  # index >= 2^bits


def test_quantize_matches_oracle_random(F, orc):
    rng = np.random.default_rng(17)
    for bits in (2, 3, 4):
        for group in (32, 128, 256):
            w = (rng.standard_normal((512, 96)) * rng.uniform(0.01, 100)).astype(np.float32)
            a = F.quantize_matrix(w, bits, group)
            b = orc.quantize(w, bits, group)
            assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
