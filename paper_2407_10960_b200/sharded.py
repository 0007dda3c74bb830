"""N-column sharding of a LUT-quantized linear layer over the GPUs of one node
(BASELINE.json configs[3]: LLaMA-3-70B K=8192, N=28672 at
1/2/4/8 GPUs).

Y = X * W_hat has independent columns, so rank r of `world` owns the 64-column
tiles [r*T/world, (r+1)*T/world) of W (columns [n0, n1), ``shard_range``).  X is
replicated (it is the previous layer's gathered output); there is no K split and
no reduction.  The only exchange is the output all-gather, done one of two ways:

* ``mode="nccl"``  — local GEMM into a [m][n1-n0] slice, then
  ``all_gather_into_tensor`` (NCCL over NVLink / NVSwitch) and a column
  re-layout for m > 1 (the gather is shard-major [P][m][N/P]).
* ``mode="peer"``  — the all-gather fused into the GEMM epilogue: every rank's
  kernel stores its column slice straight into every rank's full Y through
  symmetric-memory peer pointers (``flute_gemm_peers``), followed by one
  cross-rank barrier.  No separate collective launch.

Because device-layout units are n-tile major, a shard's packed weights and
scales are contiguous byte ranges of the full device buffers, so a shard can be
cut from a full device-layout upload as well as packed from its own columns
(tests check both are identical).
"""
from __future__ import annotations

from typing import List, Sequence

import numpy as np

from . import DeviceWeights, InputError, ShardRange, shard_range


def shard_columns(indices: np.ndarray, scales: np.ndarray, group: int, r: ShardRange):
    """Column slice [n0, n1) of an index matrix [k][n] and its [n][k/g] scales."""
    k, n = indices.shape
    sc = np.ascontiguousarray(scales, np.uint16).reshape(n, k // group)
    return (np.ascontiguousarray(indices[:, r.n0:r.n1]),
            np.ascontiguousarray(sc[r.n0:r.n1]).reshape(-1))


def gather_columns(y_local, ranges: Sequence[ShardRange], n: int, group=None):
    """All-gather the ranks' [m][n1-n0] column slices into the full [m][n].

    Works with any torch.distributed backend (NCCL on GPUs, gloo on CPU for the
    host-logic tests).  Slices are padded to the widest shard so the collective
    is a single ``all_gather_into_tensor``; the result is shard-major
    [P][m][w] and is re-laid out into columns."""
    import torch
    import torch.distributed as dist

    world = len(ranges)
    m = y_local.shape[0]
    w = max(r.n1 - r.n0 for r in ranges)
    if y_local.shape[1] < w:
        pad = torch.zeros((m, w), dtype=y_local.dtype, device=y_local.device)
        pad[:, :y_local.shape[1]] = y_local
        y_local = pad
    buf = torch.empty((world, m, w), dtype=y_local.dtype, device=y_local.device)
    if world == 1:
        buf[0].copy_(y_local)
    elif y_local.device.type == "cpu" and dist.get_backend(group) == "gloo":
        dist.all_gather(list(buf.unbind(0)), y_local.contiguous(), group=group)
    else:
        dist.all_gather_into_tensor(buf, y_local.contiguous(), group=group)
    if m == 1 and all(r.n1 - r.n0 == w for r in ranges):
        return buf.reshape(1, world * w)[:, :n]  # shard-major == row-major for one row
    out = torch.empty((m, n), dtype=y_local.dtype, device=y_local.device)
    for i, r in enumerate(ranges):
        out[:, r.n0:r.n1] = buf[i, :, :r.n1 - r.n0]
    return out


class ShardedWeights:
    """This rank's column shard of a LUT-quantized [k][n] weight matrix."""

    def __init__(self, indices: np.ndarray, scales: np.ndarray, table_values: np.ndarray,
                 bits: int, group: int, rank: int, world: int, pg=None, mode: str = "nccl"):
        if mode not in ("nccl", "peer"):
            raise InputError("mode must be 'nccl' or 'peer'")
        self.k, self.n = indices.shape
        self.bits, self.group = bits, group
        self.rank, self.world, self.pg, self.mode = rank, world, pg, mode
        self.ranges: List[ShardRange] = [shard_range(self.k, self.n, bits, group, world, r)
                                         for r in range(world)]
        self.range = self.ranges[rank]
        idx, sc = shard_columns(indices, scales, group, self.range)
        self.local = DeviceWeights(idx, sc, table_values, bits, group)
        self._symm = {}  # m -> (tensor, handle)

    # -- NCCL path -------------------------------------------------------------
    def gemm(self, x, workers: int = 0):
        """Full Y [m][n] on every rank (x: this rank's cuda f16 [m][k])."""
        if self.mode == "peer":
            return self.gemm_peer(x, workers)
        y_local = self.local.gemm(x, workers=workers)
        return gather_columns(y_local, self.ranges, self.n, self.pg)

    # -- fused peer-store path ---------------------------------------------------
    def _symm_buffer(self, m: int):
        if m not in self._symm:
            import torch
            import torch.distributed as dist
            import torch.distributed._symmetric_memory as symm_mem
            t = symm_mem.empty((m, self.n), dtype=torch.float16, device=f"cuda:{torch.cuda.current_device()}")
            h = symm_mem.rendezvous(t, self.pg if self.pg is not None else dist.group.WORLD)
            self._symm[m] = (t, h)
        return self._symm[m]

    def gemm_peer(self, x, workers: int = 0):
        """Fused all-gather: the epilogue writes this rank's columns into every
        rank's symmetric Y buffer; one barrier makes the full Y visible.

        The returned tensor ALIASES the internal symmetric buffer for this m:
        it is valid until the next gemm_peer call with the same m (which
        overwrites it).  Copy it (``.clone()``) to keep a result."""
        t, h = self._symm_buffer(x.shape[0])
        ptrs = [int(p) for p in h.buffer_ptrs]
        h.barrier()  # every rank done reading the previous contents
        self.local.gemm_peers(x, ptrs, ldy=self.n, ycol0=self.range.n0, workers=workers)
        h.barrier()  # every rank's slice has landed everywhere
        return t

    @staticmethod
    def gemm_peers_local(shards: Sequence["ShardedWeights"], x, outputs: Sequence,
                         workers: int = 0) -> None:
        """Single-process emulation of the fused path (all shards on one GPU,
        every output buffer on that GPU): used by the parity tests."""
        ptrs = [int(o.data_ptr()) for o in outputs]
        for s in shards:
            s.local.gemm_peers(x, ptrs, ldy=s.n, ycol0=s.range.n0, workers=workers)


# ---------------------------------------------------------------------------
# C++ host path (include/flutesim/sharded.hpp via the C ABI): NCCL loaded by the
# library itself, fused path over CUDA IPC peer mappings + a device flag barrier
# ---------------------------------------------------------------------------

class NcclComm:
    """flute_comm: one NCCL communicator owned by the C++ library.  The 128-byte
    unique id is created on rank 0 and broadcast over an existing
    torch.distributed group (any backend)."""

    def __init__(self, rank: int, world: int, pg=None):
        import ctypes as C
        import torch.distributed as dist
        from . import _check, _lib
        self.rank, self.world = rank, world
        uid = np.zeros(128, np.uint8)
        if rank == 0:
            _check(_lib.flute_comm_unique_id(uid))
        if world > 1:
            obj = [uid.tobytes()]
            dist.broadcast_object_list(obj, src=0, group=pg)
            uid = np.frombuffer(obj[0], np.uint8).copy()
        h = C.c_void_p()
        _check(_lib.flute_comm_create(uid, world, rank, C.byref(h)))
        self._h = h

    def close(self):
        from . import _lib
        if getattr(self, "_h", None):
            _lib.flute_comm_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class NativeShardedWeights:
    """flute_sharded: this rank's column shard, C++ host side.  ``gemm`` =
    shard GEMM + ncclAllGather + re-layout; ``gemm_fused`` = peer-store
    epilogue into every rank's double-buffered arena + device flag barrier
    (the returned tensor aliases the arena: valid until the call after next)."""

    def __init__(self, comm: NcclComm, indices: np.ndarray, scales: np.ndarray,
                 table_values: np.ndarray, bits: int, group: int, max_m: int = 32):
        import ctypes as C
        from . import _check, _lib
        idx = np.ascontiguousarray(indices, np.uint8)
        self.k, self.n = idx.shape
        self.bits, self.group, self.max_m, self.comm = bits, group, max_m, comm
        h = C.c_void_p()
        _check(_lib.flute_sharded_create(comm._h, idx, np.ascontiguousarray(scales, np.uint16),
                                         np.ascontiguousarray(table_values, np.float32), self.k,
                                         self.n, bits, group, max_m, C.byref(h)))
        self._h = h
        n0, n1 = C.c_int(0), C.c_int(0)
        _check(_lib.flute_sharded_info(h, C.byref(n0), C.byref(n1)))
        self.n0, self.n1 = n0.value, n1.value

    def _check_x(self, x):
        import torch
        if x.dtype != torch.float16 or not x.is_cuda or x.dim() != 2 or x.shape[1] != self.k:
            raise InputError(f"x must be a cuda float16 [m][{self.k}] tensor")
        return x.contiguous()

    def gemm(self, x, y=None, stream=None):
        import torch
        from . import _check, _lib, _stream_ptr
        x = self._check_x(x)
        if y is None:
            y = torch.empty((x.shape[0], self.n), dtype=torch.float16, device=x.device)
        elif (y.dtype != torch.float16 or y.device != x.device or tuple(y.shape) != (x.shape[0], self.n)
              or not y.is_contiguous()):
            raise InputError(f"y must be a contiguous float16 [{x.shape[0]}][{self.n}] tensor on {x.device}")
        _check(_lib.flute_sharded_gemm(self._h, x.data_ptr(), x.shape[0], y.data_ptr(),
                                       _stream_ptr(stream)))
        return y

    def gemm_fused(self, x, stream=None):
        """Full Y as a [m][n] view of the library's arena (no copy)."""
        import ctypes as C
        from . import _check, _lib, _stream_ptr
        x = self._check_x(x)
        m = x.shape[0]
        out = C.c_void_p()
        _check(_lib.flute_sharded_gemm_fused(self._h, x.data_ptr(), m, C.byref(out),
                                             _stream_ptr(stream)))
        # wrap the arena pointer (lifetime = this object) without a copy
        return _wrap_device_f16(out.value, (m, self.n), x.device)

    def close(self):
        from . import _lib
        if getattr(self, "_h", None):
            _lib.flute_sharded_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _wrap_device_f16(ptr: int, shape, device):
    """A torch view of an f16 device buffer owned by the library."""
    import torch

    class _Arr:
        __cuda_array_interface__ = {"shape": tuple(shape), "typestr": "<f2", "data": (ptr, False),
                                    "version": 3, "strides": None}
    return torch.as_tensor(_Arr(), device=device)


def shard_from_device_layout(full_packed: np.ndarray, full_scales_dev: np.ndarray, r: ShardRange):
    """Cut a shard's device-layout weights / scales out of the full buffers
    (contiguous byte ranges; pure slicing, no re-pack)."""
    w = np.ascontiguousarray(full_packed[r.w_off:r.w_off + r.w_bytes])
    s = np.ascontiguousarray(full_scales_dev.view(np.uint8)[r.s_off:r.s_off + r.s_bytes]).view(np.uint16)
    return w, s


def make_shards_single_process(indices, scales, table_values, bits, group, world,
                               mode: str = "nccl") -> List[ShardedWeights]:
    """All `world` shards in one process (one GPU): the parity tests' stand-in
    for a multi-GPU run."""
    out = []
    for r in range(world):
        s = ShardedWeights.__new__(ShardedWeights)
        s.k, s.n = indices.shape
        s.bits, s.group, s.rank, s.world, s.pg, s.mode = bits, group, r, world, None, mode
        s.ranges = [shard_range(s.k, s.n, bits, group, world, i) for i in range(world)]
        s.range = s.ranges[r]
        idx, sc = shard_columns(indices, scales, group, s.range)
        s.local = DeviceWeights(idx, sc, table_values, bits, group)
        s._symm = {}
        out.append(s)
    return out


__all__ = ["ShardedWeights", "NativeShardedWeights", "NcclComm", "gather_columns", "shard_columns",
           "shard_from_device_layout", "make_shards_single_process"]
