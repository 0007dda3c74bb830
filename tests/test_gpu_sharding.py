"""GPU half of the N-column sharding tests: every shard's
GEMM through the product kernel, concatenated, matches the full layer; the
fused peer-store all-gather writes identical full outputs into every rank's
buffer.  Multi-GPU ranks are emulated on one GPU (all peers' buffers on the
same device; the kernel path is identical for NVLink peer pointers)."""
import numpy as np
import pytest

from conftest import f16_bits

pytestmark = pytest.mark.gpu


def _layer(F, orc, rng, m, k, n, bits, group):
    w = rng.standard_normal((k, n)).astype(np.float32)
    idx, scales = F.quantize_matrix(w, bits, group)
    table = F.build_nf_table(bits)
    x16 = f16_bits(orc, rng.standard_normal((m, k)) * 0.5)
    y64 = orc.reference_f64(x16, idx, bits, group, scales, table)
    return idx, scales, table, x16, y64


def _within(y16, y64, tol=1e-2):
    y = y16.view(np.float16).astype(np.float64)
    bound = tol * np.maximum(np.abs(y64), np.sqrt(np.mean(y64 ** 2)) + 1e-30)
    return bool(np.all(np.abs(y - y64) <= bound))


@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("m", [1, 5])
def test_sharded_columns_match_full_layer(F, orc, gpu, world, m):
    from paper_2407_10960_b200.sharded import make_shards_single_process
    rng = np.random.default_rng(world * 10 + m)
    k, n, bits, group = 1024, 1024, 4, 128
    idx, scales, table, x16, y64 = _layer(F, orc, rng, m, k, n, bits, group)
    shards = make_shards_single_process(idx, scales, table, bits, group, world)
    x = gpu.from_numpy(x16.view(np.float16)).cuda()
    parts = [s.local.gemm(x) for s in shards]
    y = gpu.cat(parts, dim=1).cpu().numpy().view(np.uint16)
    assert y.shape == (m, n)
    assert _within(y, y64)


@pytest.mark.parametrize("world,m,bits", [(2, 1, 4), (4, 3, 3), (8, 1, 4), (8, 17, 2)])
def test_fused_peer_allgather(F, orc, gpu, world, m, bits):
    """Each shard's epilogue stores its columns into all `world` full-size
    outputs; after all shards ran, every output holds the same full Y."""
    from paper_2407_10960_b200.sharded import ShardedWeights, make_shards_single_process
    rng = np.random.default_rng(100 + world + m + bits)
    k, n, group = 512, 2048, 64
    idx, scales, table, x16, y64 = _layer(F, orc, rng, m, k, n, bits, group)
    shards = make_shards_single_process(idx, scales, table, bits, group, world, mode="peer")
    x = gpu.from_numpy(x16.view(np.float16)).cuda()
    outs = [gpu.full((m, n), float("nan"), dtype=gpu.float16, device="cuda") for _ in range(world)]
    ShardedWeights.gemm_peers_local(shards, x, outs)
    gpu.cuda.synchronize()
    ys = [o.cpu().numpy().view(np.uint16) for o in outs]
    for y in ys[1:]:
        assert np.array_equal(y, ys[0])
    assert _within(ys[0], y64)
    # same bits as the non-fused shard GEMMs
    ref = gpu.cat([s.local.gemm(x) for s in shards], dim=1).cpu().numpy().view(np.uint16)
    assert np.array_equal(ys[0], ref)


def test_peer_output_errors(F, gpu):
    rng = np.random.default_rng(3)
    idx, sc = F.quantize_matrix(rng.standard_normal((256, 128)).astype(np.float32), 4, 128)
    dw = F.DeviceWeights(idx, sc, F.build_nf_table(4), 4, 128)
    x = gpu.zeros((1, 256), dtype=gpu.float16, device="cuda")
    y = gpu.zeros((1, 128), dtype=gpu.float16, device="cuda")
    with pytest.raises(F.ConfigError):
        dw.gemm_peers(x, [y.data_ptr()] * 9, ldy=128, ycol0=0)
    with pytest.raises(F.ConfigError):
        dw.gemm_peers(x, [y.data_ptr()], ldy=100, ycol0=0)  # ldy < ycol0 + n
    with pytest.raises(F.InputError):
        dw.gemm_peers(x, [0], ldy=128, ycol0=0)


def test_sharded_weights_world1_nccl(F, orc, gpu):
    """The public ShardedWeights API end to end on a real (1-rank) NCCL group."""
    import os
    import socket
    import torch.distributed as dist
    from paper_2407_10960_b200.sharded import ShardedWeights
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=gpu.device("cuda", 0))
    try:
        rng = np.random.default_rng(9)
        idx, scales, table, x16, y64 = _layer(F, orc, rng, 2, 512, 256, 4, 128)
        sw = ShardedWeights(idx, scales, table, 4, 128, rank=0, world=1)
        y = sw.gemm(gpu.from_numpy(x16.view(np.float16)).cuda())
        assert _within(y.cpu().numpy().view(np.uint16), y64)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("m", [1, 5])
def test_native_sharded_world1(F, gpu, m):
    """The C++ sharded layer (flute_sharded_*: NCCL loaded by the library,
    fused peer-store + device flag barrier) at world 1 on the one GPU: both
    paths equal the plain device GEMM bitwise, repeatedly (the fused path's
    double-buffered arena alternates and stays correct)."""
    from paper_2407_10960_b200.sharded import NativeShardedWeights, NcclComm
    rng = np.random.default_rng(77 + m)
    k, n, bits, group = 1024, 512, 4, 128
    idx, sc = F.quantize_matrix(rng.standard_normal((k, n)).astype(np.float32), bits, group)
    table = F.build_nf_table(bits)
    comm = NcclComm(0, 1)
    sw = NativeShardedWeights(comm, idx, sc, table, bits, group, max_m=8)
    assert (sw.n0, sw.n1) == (0, n)
    dw = F.DeviceWeights(idx, sc, table, bits, group)
    for it in range(4):
        x = (gpu.randn(m, k, device="cuda") * 0.5).half()
        want = dw.gemm(x).cpu()
        got = sw.gemm(x).cpu()
        fused = sw.gemm_fused(x).clone().cpu()
        gpu.cuda.synchronize()
        assert gpu.equal(got.view(gpu.int16), want.view(gpu.int16)), it
        assert gpu.equal(fused.view(gpu.int16), want.view(gpu.int16)), it
    with pytest.raises(F.ConfigError):
        sw.gemm_fused((gpu.randn(9, k, device="cuda")).half())  # m > max_m
    sw.close()
    comm.close()
