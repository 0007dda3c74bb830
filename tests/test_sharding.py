"""N-column sharding: shard geometry, device-layout
contiguity, and the all-gather + column re-layout over a real 2-process gloo
group on CPU.  The GPU halves (each shard's GEMM, the fused peer-store
all-gather) are in test_gpu_sharding.py."""
import os
import socket

import numpy as np
import pytest

from conftest import f16_bits


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_shard_range_70b_layer(F, world):
    """configs[3]: K=8192, N=28672 W4 g128 — equal 64-aligned column slices,
    contiguous device-layout byte ranges that tile the full buffers."""
    k, n, bits, group = 8192, 28672, 4, 128
    wb, sb = F.device_sizes(k, n, bits, group)
    rs = [F.shard_range(k, n, bits, group, world, r) for r in range(world)]
    assert rs[0].n0 == 0 and rs[-1].n1 == n
    for a, b in zip(rs, rs[1:]):
        assert a.n1 == b.n0 and a.w_off + a.w_bytes == b.w_off and a.s_off + a.s_bytes == b.s_off
    assert all(r.n0 % 64 == 0 and r.n1 - r.n0 == n // world for r in rs)
    assert sum(r.w_bytes for r in rs) == wb and sum(r.s_bytes for r in rs) == sb
    # per-GPU algorithmic bytes at P = 8 (15.2 MB)
    if world == 8:
        assert abs(rs[0].w_bytes + rs[0].s_bytes - 15.1e6) < 0.2e6


def test_shard_range_errors(F):
    with pytest.raises(F.ConfigError):
        F.shard_range(256, 128, 4, 128, 3, 0)  # 2 tiles, 3 ranks
    with pytest.raises(F.ConfigError):
        F.shard_range(256, 128, 4, 128, 2, 2)


@pytest.mark.parametrize("bits", [2, 3, 4])
@pytest.mark.parametrize("k,n,group,world", [(256, 320, 64, 2), (384, 448, 128, 3), (512, 256, 32, 4)])
def test_shard_is_contiguous_slice_of_device_layout(F, bits, k, n, group, world):
    """Packing a shard's own columns == slicing the full device-layout upload."""
    from paper_2407_10960_b200.sharded import shard_columns, shard_from_device_layout
    rng = np.random.default_rng(bits * 100 + world)
    idx, sc = F.quantize_matrix(rng.standard_normal((k, n)).astype(np.float32), bits, group)
    full_w = F.pack_device(idx, bits, group)
    full_s = F.scales_device(sc, k, n, group)
    for r in range(world):
        rr = F.shard_range(k, n, bits, group, world, r)
        i_s, s_s = shard_columns(idx, sc, group, rr)
        w_cut, s_cut = shard_from_device_layout(full_w, full_s, rr)
        assert np.array_equal(F.pack_device(i_s, bits, group), w_cut)
        assert np.array_equal(F.scales_device(s_s, k, rr.n1 - rr.n0, group), s_cut)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _gloo_worker(rank, world, port, m, k, n, result_q):
    import torch
    import torch.distributed as dist
    import paper_2407_10960_b200 as F
    from paper_2407_10960_b200.sharded import gather_columns
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(1234)  # same data on every rank
        w = rng.standard_normal((k, n)).astype(np.float32)
        x = rng.standard_normal((m, k)).astype(np.float32)
        ranges = [F.shard_range(k, n, 4, 128, world, r) for r in range(world)]
        me = ranges[rank]
        y_local = torch.from_numpy(x @ w[:, me.n0:me.n1])  # stand-in for the shard GEMM
        y = gather_columns(y_local, ranges, n)
        ok = bool(np.allclose(y.numpy(), x @ w, rtol=1e-5, atol=1e-4))
        result_q.put((rank, ok, tuple(y.shape)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("m,n", [(1, 512), (3, 448)])
def test_gather_columns_gloo_world2(m, n):
    """Real 2-process gloo group: each rank's column slice all-gathered and
    re-laid out equals the full product (m = 1 takes the shard-major fast
    path, m > 1 / uneven shards the re-layout)."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    k = 256
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, m, k, n, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert sorted(r[0] for r in res) == [0, 1]
    assert all(ok for _, ok, _ in res), res
    assert all(shape == (m, n) for _, _, shape in res)


def _gloo_shard_worker(rank, world, port, m, k, n, bits, group, result_q):
    """One rank of the sharded layer with the product's host-side shard path
    (shard_range -> shard_columns -> the shard's own canonical packing) and
    the CPU oracle's engine standing in for the shard's device GEMM (test
    infrastructure; the device GEMM is test_gpu_sharding.py)."""
    import torch
    import torch.distributed as dist
    import paper_2407_10960_b200 as F
    from oracle import Oracle
    from paper_2407_10960_b200.sharded import gather_columns, shard_columns
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        orc = Oracle()
        rng = np.random.default_rng(4242)  # same full matrix on every rank
        idx, sc = F.quantize_matrix(rng.standard_normal((k, n)).astype(np.float32), bits, group)
        table = F.build_nf_table(bits)
        x16 = (rng.standard_normal((m, k)) * 0.5).astype(np.float16).view(np.uint16)
        ranges = [F.shard_range(k, n, bits, group, world, r) for r in range(world)]
        me = ranges[rank]
        i_s, s_s = shard_columns(idx, sc, group, me)
        w = me.n1 - me.n0
        y_s, _ = orc.execute(x16, orc.pack(i_s, bits), k, w, bits, group, s_s, table, workers=1)
        # (gloo has no 16-bit integer type: the f16 bit patterns travel as int32)
        y = gather_columns(torch.from_numpy(y_s.astype(np.int32)), ranges, n)
        y_full, _ = orc.execute(x16, orc.pack(idx, bits), k, n, bits, group, sc, table, workers=1)
        ok = bool(np.array_equal(y.numpy().astype(np.uint16), y_full))
        result_q.put((rank, ok, tuple(y.shape)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("m,n,bits", [(1, 512, 4), (3, 448, 3)])
def test_sharded_layer_gloo_world2_bitwise(m, n, bits):
    """The column-sharded layer over a real 2-process gloo group: every rank's
    shard (cut by the product's host code) computed by the reference engine's
    restatement, all-gathered and re-laid out, equals the unsharded engine
    output BITWISE (columns are independent; with one worker the per-tile k
    order is the same) — the N-sharding contract of SURVEY.md §8(e)."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    k, group = 256, 64
    procs = [ctx.Process(target=_gloo_shard_worker, args=(r, 2, port, m, k, n, bits, group, q))
             for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert sorted(r[0] for r in res) == [0, 1]
    assert all(ok for _, ok, _ in res), res
    assert all(shape == (m, n) for _, _, shape in res)
