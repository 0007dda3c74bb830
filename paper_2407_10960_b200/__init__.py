"""flute-b200 — B200-native LUT-quantized GEMM (FLUTE, arXiv 2407.10960).

Python front-end over the C ABI in ``include/flute_c.h`` (the product is the
C++/CUDA library ``libflute_b200.so`` next to this file).  Names follow the
reference C++ API (``reorder_and_split``, ``make_vectorized_lut``,
``plan_stream_k``, ``execute`` …; reference: /root/reference/proj/include/
flutesim/*.hpp) so that tests read like the reference's own.

There is no CPU fallback: GPU entry points raise :class:`CudaError` when the
library or an sm_100 device is unavailable, and importing this package fails
loudly if the shared library has not been built (``__graft_entry__.build()``).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FLUTE_LIB") or os.path.join(_HERE, "libflute_b200.so")

DEFAULT_LAYOUT = (16, 64, 64, 16, 8, 16)  # reference pack.hpp:21-26
UNIT_N, UNIT_K = 64, 128                  # device Stream-K unit (pack.hpp kUnitN/kUnitK)


class FluteError(RuntimeError):
    code = 0


class ConfigError(FluteError):
    code = 1


class InputError(FluteError):
    code = 2


class InternalError(FluteError):
    code = 3


class CudaError(FluteError):
    code = 4


class OptimizationError(FluteError):
    """refine_scales' loss or folded scale went non-finite (errors.hpp
    OptimizationError); .step is the failing step."""
    code = 5
    step = -1


_ERRS = {1: ConfigError, 2: InputError, 3: InternalError, 4: CudaError, 5: OptimizationError}


def build(force: bool = False) -> str:
    """Compile the product library in-tree (nvcc for sm_100a + g++)."""
    if force:
        subprocess.run(["make", "-s", "-C", os.path.join(_HERE, "csrc"), "clean"], check=True)
    subprocess.run(["make", "-s", "-j8", "-C", os.path.join(_HERE, "csrc")], check=True)
    return LIB_PATH


def _load() -> C.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
            " (there is no CPU fallback)")
    return C.CDLL(LIB_PATH)


_lib = _load()

_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_u16p = np.ctypeslib.ndpointer(np.uint16, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_vp = C.c_void_p

# Every symbol include/flute_c.h declares, with its ctypes signature.
_SIGS = {
    "flute_last_error": (C.c_char_p, []),
    "flute_version": (C.c_char_p, []),
    "flute_f32_to_f16": (C.c_uint16, [C.c_float]),
    "flute_f16_to_f32": (C.c_float, [C.c_uint16]),
    "flute_nf_table": (C.c_int, [C.c_int, _f32p]),
    "flute_nf_quantiles": (C.c_int, [C.c_int, _f64p]),
    "flute_nf_sigma": (C.c_double, []),
    "flute_quantize": (C.c_int, [_f32p, C.c_int, C.c_int, C.c_int, C.c_int, _u8p, _u16p]),
    "flute_canonical_words": (C.c_size_t, [C.c_int, C.c_int, C.c_int]),
    "flute_pack_canonical": (C.c_int, [_u8p, C.c_int, C.c_int, C.c_int, _i32p, _u32p, _vp]),
    "flute_unpack_canonical": (C.c_int, [_u32p, _vp, C.c_int, C.c_int, C.c_int, _i32p, _u8p]),
    "flute_device_sizes": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int,
                                     C.POINTER(C.c_size_t), C.POINTER(C.c_size_t)]),
    "flute_pack_device": (C.c_int, [_u8p, C.c_int, C.c_int, C.c_int, C.c_int, _u8p]),
    "flute_repack_canonical": (C.c_int, [_u32p, _vp, C.c_int, C.c_int, C.c_int, _i32p, C.c_int,
                                         _u8p]),
    "flute_unpack_device": (C.c_int, [_u8p, C.c_int, C.c_int, C.c_int, C.c_int, _u8p]),
    "flute_scales_device": (C.c_int, [_u16p, C.c_int, C.c_int, C.c_int, _u16p]),
    "flute_vlut_build": (C.c_int, [_f32p, C.c_int, C.c_int, _u32p]),
    "flute_vlut_device_words": (C.c_int, [_u32p, C.c_int, _u32p]),
    "flute_vec_dequantize": (C.c_int, [C.c_uint32, C.c_uint16, _u32p, C.c_int,
                                       C.POINTER(C.c_uint32)]),
    "flute_plan_stream_k": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, _i64p, _vp, C.c_int,
                                      C.POINTER(C.c_int), C.POINTER(C.c_int64)]),
    "flute_plan_traffic": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _i32p, C.c_int,
                                     C.c_int, C.c_int, _u64p]),
    "flute_bits_per_param": (C.c_double, [C.c_int, C.c_int]),
    "flute_device_count": (C.c_int, []),
    "flute_sm_count": (C.c_int, [C.c_int]),
    "flute_max_workers": (C.c_int, [C.c_int]),
    "flute_default_workers": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int]),
    "flute_workspace_bytes": (C.c_size_t, [C.c_int, C.c_int]),
    "flute_qgemm": (C.c_int, [_vp, C.c_int, C.c_int, C.c_int, _vp, _vp, _vp, C.c_int, C.c_int,
                              _vp, _vp, C.c_size_t, C.c_int, _vp]),
    "flute_weights_create": (C.c_int, [_u8p, _u16p, _u32p, C.c_int, C.c_int, C.c_int, C.c_int,
                                       C.POINTER(_vp)]),
    "flute_weights_from_indices": (C.c_int, [_u8p, _u16p, _f32p, C.c_int, C.c_int, C.c_int,
                                             C.c_int, C.POINTER(_vp)]),
    "flute_weights_destroy": (C.c_int, [_vp]),
    "flute_weights_reserve": (C.c_int, [_vp, C.c_int]),
    "flute_weights_autotune": (C.c_int, [_vp, C.c_int, _vp, C.c_char_p, C.c_size_t]),
    "flute_weights_info": (C.c_int, [_vp, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                     C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "flute_gemm": (C.c_int, [_vp, _vp, C.c_int, _vp, C.c_int, _vp]),
    "flute_gemm_host": (C.c_int, [_vp, _u16p, C.c_int, _u16p, C.c_int, _vp]),
    "flute_host_batch_create": (C.c_int, [C.POINTER(_vp), C.POINTER(C.c_void_p),
                                          C.POINTER(C.c_int), C.POINTER(C.c_void_p), C.c_int,
                                          C.c_int, C.POINTER(_vp)]),
    "flute_host_batch_run": (C.c_int, [_vp, _vp]),
    "flute_host_batch_destroy": (None, [_vp]),
    "flute_gemm_host_batch": (C.c_int, [C.POINTER(_vp), C.POINTER(C.c_void_p), C.POINTER(C.c_int),
                                        C.POINTER(C.c_void_p), C.c_int, C.c_int, _vp]),
    "flute_execute": (C.c_int, [_u16p, C.c_int, _u32p, _vp, C.c_int, C.c_int, C.c_int, C.c_int,
                                _i32p, _u16p, _u32p, C.c_int, C.c_int, C.c_int, C.c_int, _u16p,
                                _u64p]),
    "flute_quantize_device": (C.c_int, [_vp, C.c_int, C.c_int, C.c_int, C.c_int, _vp, _vp, _vp]),
    "flute_weights_from_device": (C.c_int, [_vp, _vp, _u16p, C.c_int, C.c_int, C.c_int, C.c_int,
                                            _vp, C.POINTER(_vp)]),
    "flute_flte_info": (C.c_int, [_u8p, C.c_size_t, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                  C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "flute_weights_from_flte": (C.c_int, [_u8p, C.c_size_t, _vp, C.POINTER(_vp)]),
    "flute_flte_write": (C.c_int, [_u8p, _u16p, _f32p, C.c_int, C.c_int, C.c_int, C.c_int, _i32p,
                                   _vp, C.c_size_t, C.POINTER(C.c_size_t)]),
    "flute_ste_evaluate": (C.c_int, [_f32p, _f32p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                     _f64p, C.POINTER(C.c_double), _f64p, _u8p]),
    "flute_refine_scales": (C.c_int, [_f32p, _f32p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                      C.c_int, C.c_double, _u8p, _u16p, _f64p, _f64p,
                                      C.POINTER(C.c_int)]),
    "flute_shard_range": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                    C.POINTER(C.c_int), C.POINTER(C.c_int),
                                    C.POINTER(C.c_size_t), C.POINTER(C.c_size_t),
                                    C.POINTER(C.c_size_t), C.POINTER(C.c_size_t)]),
    "flute_qgemm_peers": (C.c_int, [_vp, C.c_int, C.c_int, C.c_int, _vp, _vp, _vp, C.c_int,
                                    C.c_int, C.POINTER(C.c_void_p), C.c_int, C.c_int, C.c_int,
                                    _vp, C.c_size_t, C.c_int, _vp]),
    "flute_gemm_peers": (C.c_int, [_vp, _vp, C.c_int, C.POINTER(C.c_void_p), C.c_int, C.c_int,
                                   C.c_int, C.c_int, _vp]),
    "flute_comm_unique_id": (C.c_int, [_u8p]),
    "flute_comm_create": (C.c_int, [_u8p, C.c_int, C.c_int, C.POINTER(_vp)]),
    "flute_comm_destroy": (C.c_int, [_vp]),
    "flute_sharded_create": (C.c_int, [_vp, _u8p, _u16p, _f32p, C.c_int, C.c_int, C.c_int, C.c_int,
                                       C.c_int, C.POINTER(_vp)]),
    "flute_sharded_destroy": (C.c_int, [_vp]),
    "flute_sharded_info": (C.c_int, [_vp, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "flute_sharded_gemm": (C.c_int, [_vp, _vp, C.c_int, _vp, _vp]),
    "flute_sharded_gemm_fused": (C.c_int, [_vp, _vp, C.c_int, C.POINTER(_vp), _vp]),
    "flute_dequant_all_device": (C.c_int, [_u32p, C.c_int, _u16p, C.c_int, _u32p]),
    "flute_mma_fragment": (C.c_int, [_u16p, _u16p, _f32p, C.c_int, C.c_int, C.c_int]),
    "flute_debug_times": (C.c_int, [_u64p, C.c_int]),
}

for _name, (_res, _args) in _SIGS.items():
    _fn = getattr(_lib, _name)  # AttributeError here = a declared symbol is not exported
    _fn.restype = _res
    _fn.argtypes = _args


def _check(rc: int) -> None:
    if rc != 0:
        raise _ERRS.get(rc, FluteError)(_lib.flute_last_error().decode())


def _lay(layout) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(layout, np.int32))


def version() -> str:
    return _lib.flute_version().decode()


# --------------------------------------------------------------------------
# numerics + input producers
# --------------------------------------------------------------------------

def f32_to_f16(x: float) -> int:
    return int(_lib.flute_f32_to_f16(float(x)))


def f16_to_f32(h: int) -> float:
    return float(_lib.flute_f16_to_f32(int(h)))


def build_nf_table(bits: int) -> np.ndarray:
    out = np.zeros(1 << bits, np.float32)
    _check(_lib.flute_nf_table(bits, out))
    return out


def quantize_matrix(w: np.ndarray, bits: int, group: int):
    """quantize.hpp:45 — returns (indices u8 [k][n], scales u16 [n][k/g])."""
    w = np.ascontiguousarray(w, np.float32)
    k, n = w.shape
    idx = np.zeros((k, n), np.uint8)
    sc = np.zeros(k * n // max(group, 1), np.uint16)
    _check(_lib.flute_quantize(w, k, n, bits, group, idx, sc))
    return idx, sc


# --------------------------------------------------------------------------
# packers
# --------------------------------------------------------------------------

def canonical_words(k: int, n: int, slice_bits: int) -> int:
    return int(_lib.flute_canonical_words(k, n, slice_bits))


def reorder_and_split(indices: np.ndarray, bits: int, layout=DEFAULT_LAYOUT):
    """pack.hpp:72 — canonical slices (hi[, lo]) as u32 arrays."""
    idx = np.ascontiguousarray(indices, np.uint8)
    k, n = idx.shape
    hi = np.zeros(max(1, canonical_words(k, n, 2 if bits == 3 else bits)), np.uint32)
    lo = np.zeros(max(1, canonical_words(k, n, 1)), np.uint32) if bits == 3 else None
    _check(_lib.flute_pack_canonical(idx, k, n, bits, _lay(layout), hi,
                                     lo.ctypes.data if lo is not None else None))
    return (hi, lo) if bits == 3 else (hi,)


def unpack_matrix(slices, k: int, n: int, bits: int, layout=DEFAULT_LAYOUT) -> np.ndarray:
    hi = np.ascontiguousarray(slices[0], np.uint32)
    lo = np.ascontiguousarray(slices[1], np.uint32) if bits == 3 else None
    out = np.zeros((k, n), np.uint8)
    _check(_lib.flute_unpack_canonical(hi, lo.ctypes.data if lo is not None else None, k, n, bits,
                                       _lay(layout), out))
    return out


def device_sizes(k: int, n: int, bits: int, group: int):
    wb, sb = C.c_size_t(0), C.c_size_t(0)
    _check(_lib.flute_device_sizes(k, n, bits, group, C.byref(wb), C.byref(sb)))
    return wb.value, sb.value


def pack_device(indices: np.ndarray, bits: int, group: int) -> np.ndarray:
    idx = np.ascontiguousarray(indices, np.uint8)
    k, n = idx.shape
    wb, _ = device_sizes(k, n, bits, group)
    out = np.zeros(wb, np.uint8)
    _check(_lib.flute_pack_device(idx, k, n, bits, group, out))
    return out


def repack_canonical(slices, k: int, n: int, bits: int, group: int, layout=DEFAULT_LAYOUT):
    hi = np.ascontiguousarray(slices[0], np.uint32)
    lo = np.ascontiguousarray(slices[1], np.uint32) if bits == 3 else None
    wb, _ = device_sizes(k, n, bits, group)
    out = np.zeros(wb, np.uint8)
    _check(_lib.flute_repack_canonical(hi, lo.ctypes.data if lo is not None else None, k, n, bits,
                                       _lay(layout), group, out))
    return out


def unpack_device(packed: np.ndarray, k: int, n: int, bits: int, group: int) -> np.ndarray:
    out = np.zeros((k, n), np.uint8)
    _check(_lib.flute_unpack_device(np.ascontiguousarray(packed, np.uint8), k, n, bits, group,
                                    out))
    return out


def scales_device(scales: np.ndarray, k: int, n: int, group: int) -> np.ndarray:
    _, sb = device_sizes(k, n, 4, group)
    out = np.zeros(sb // 2, np.uint16)
    _check(_lib.flute_scales_device(np.ascontiguousarray(scales, np.uint16), k, n, group, out))
    return out


# --------------------------------------------------------------------------
# vLUT
# --------------------------------------------------------------------------

def make_vectorized_lut(table_values: np.ndarray, bits: int, dup: int = 1) -> np.ndarray:
    """vec_lut.hpp:34 — 2^(2b)*dup u32 words (first | second << 16)."""
    out = np.zeros((1 << (2 * bits)) * max(dup, 1), np.uint32)
    _check(_lib.flute_vlut_build(np.ascontiguousarray(table_values, np.float32), bits, dup, out))
    return out


def vlut_device_words(vlut_words: np.ndarray, bits: int) -> np.ndarray:
    out = np.zeros(1 << (2 * bits), np.uint32)
    _check(_lib.flute_vlut_device_words(np.ascontiguousarray(vlut_words, np.uint32), bits, out))
    return out


def vec_dequantize(pair: int, scale: int, vlut_words: np.ndarray, bits: int) -> int:
    o = C.c_uint32(0)
    _check(_lib.flute_vec_dequantize(pair, scale, np.ascontiguousarray(vlut_words, np.uint32),
                                     bits, C.byref(o)))
    return o.value


# --------------------------------------------------------------------------
# Stream-K + traffic
# --------------------------------------------------------------------------

@dataclass
class StreamKPlan:
    ranges: np.ndarray   # [workers, 2]
    fixups: np.ndarray   # [n_fixups, 4] (tile, finisher, slot_base, n_contributors)
    total_slots: int


def plan_stream_k(tiles_m: int, tiles_n: int, tiles_k: int, workers: int) -> StreamKPlan:
    ranges = np.zeros(2 * max(workers, 1), np.int64)
    cap = max(tiles_m * tiles_n, 1)
    fx = np.zeros(4 * cap, np.int64)
    nf, slots = C.c_int(0), C.c_int64(0)
    _check(_lib.flute_plan_stream_k(tiles_m, tiles_n, tiles_k, workers, ranges, fx.ctypes.data,
                                    cap, C.byref(nf), C.byref(slots)))
    return StreamKPlan(ranges.reshape(-1, 2), fx[:4 * nf.value].reshape(-1, 4), slots.value)


TRAFFIC_FIELDS = ("bytes_weights", "bytes_scales", "bytes_table", "bytes_activations",
                  "bytes_partials_rw", "bytes_output", "flops")


def plan_traffic(m, k, n, bits, group, layout=DEFAULT_LAYOUT, workers=1, stages=2, tile_m=0):
    st = np.zeros(7, np.uint64)
    _check(_lib.flute_plan_traffic(m, k, n, bits, group, _lay(layout), workers, stages, tile_m,
                                   st))
    return dict(zip(TRAFFIC_FIELDS, (int(v) for v in st)))


def bits_per_param(bits: int, group: int) -> float:
    v = _lib.flute_bits_per_param(bits, group)
    if v < 0:
        raise ConfigError(_lib.flute_last_error().decode())
    return float(v)


def algorithmic_bytes(m: int, k: int, n: int, bits: int, group: int) -> int:
    """each byte counted once."""
    return (k * n * bits + 7) // 8 + (k * n // group) * 2 + m * k * 2 + m * n * 2 + (1 << bits) * 2


# --------------------------------------------------------------------------
# device
# --------------------------------------------------------------------------

def device_count() -> int:
    return int(_lib.flute_device_count())


def sm_count(device: int = 0) -> int:
    v = _lib.flute_sm_count(device)
    if v < 0:
        raise CudaError(_lib.flute_last_error().decode())
    return int(v)


def default_workers(m: int, k: int, n: int, bits: int) -> int:
    v = _lib.flute_default_workers(m, k, n, bits)
    if v < 0:
        raise CudaError(_lib.flute_last_error().decode())
    return int(v)


def workspace_bytes(m: int, workers: int) -> int:
    return int(_lib.flute_workspace_bytes(m, workers))


def _stream_ptr(stream) -> Optional[int]:
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    return int(stream)


class DeviceWeights:
    """Device-resident quantized weights (uploaded once).  ``gemm`` is the hot
    path: device tensors in, device tensor out, async on the current torch
    stream.  Mirrors flutesim::DeviceWeights (include/flutesim/engine.hpp)."""

    def __init__(self, indices: np.ndarray, scales: np.ndarray, table_values: np.ndarray,
                 bits: int, group: int):
        idx = np.ascontiguousarray(indices, np.uint8)
        self.k, self.n = idx.shape
        self.bits, self.group = bits, group
        h = _vp()
        _check(_lib.flute_weights_from_indices(idx, np.ascontiguousarray(scales, np.uint16),
                                               np.ascontiguousarray(table_values, np.float32),
                                               self.k, self.n, bits, group, C.byref(h)))
        self._h = h

    @classmethod
    def from_device_layout(cls, packed: np.ndarray, scales_dev: np.ndarray,
                           vlut_words: np.ndarray, k: int, n: int, bits: int, group: int):
        self = cls.__new__(cls)
        self.k, self.n, self.bits, self.group = k, n, bits, group
        h = _vp()
        _check(_lib.flute_weights_create(np.ascontiguousarray(packed, np.uint8),
                                         np.ascontiguousarray(scales_dev, np.uint16),
                                         np.ascontiguousarray(vlut_words, np.uint32), k, n, bits,
                                         group, C.byref(h)))
        self._h = h
        return self

    def reserve(self, max_m: int) -> None:
        """Pre-size the workspace for m <= max_m (no allocation in later calls,
        e.g. inside CUDA-graph capture; m <= 32 never allocates)."""
        _check(_lib.flute_weights_reserve(self._h, max_m))

    @classmethod
    def _from_handle(cls, h, k, n, bits, group):
        self = cls.__new__(cls)
        self.k, self.n, self.bits, self.group = k, n, bits, group
        self._h = h
        return self

    @classmethod
    def from_device_indices(cls, idx, scales, table16: np.ndarray, bits: int, group: int,
                            stream=None):
        """From device-resident torch tensors: idx uint8 [k][n], scales int16/
        uint16 bits [n*k/g] (e.g. quantize_matrix_device's outputs); packed into
        the device layout on the GPU."""
        k, n = idx.shape
        h = _vp()
        _check(_lib.flute_weights_from_device(idx.data_ptr(), scales.data_ptr(),
                                              np.ascontiguousarray(table16, np.uint16), k, n,
                                              bits, group, _stream_ptr(stream), C.byref(h)))
        return cls._from_handle(h, k, n, bits, group)

    @classmethod
    def from_flte(cls, data, stream=None):
        """From an FLTE container (bytes or a path): the canonical slices are
        uploaded as stored and re-permuted to the device layout on the GPU."""
        if isinstance(data, (str, os.PathLike)):
            with open(data, "rb") as f:
                data = f.read()
        buf = np.frombuffer(bytes(data), np.uint8).copy()
        bits, group, k, n = (C.c_int(0) for _ in range(4))
        _check(_lib.flute_flte_info(buf, buf.size, C.byref(bits), C.byref(group), C.byref(k),
                                    C.byref(n)))
        h = _vp()
        _check(_lib.flute_weights_from_flte(buf, buf.size, _stream_ptr(stream), C.byref(h)))
        return cls._from_handle(h, k.value, n.value, bits.value, group.value)

    def autotune(self, m: int, stream=None) -> str:
        """Time the candidate decompositions for m-row calls (L2 flushed) and
        keep the fastest for this handle's default-worker calls of that row
        class (M <= 8 / 16 / 32).  Returns the timing report."""
        buf = C.create_string_buffer(4096)
        _check(_lib.flute_weights_autotune(self._h, m, _stream_ptr(stream), buf, 4096))
        return buf.value.decode()

    def close(self) -> None:
        if getattr(self, "_h", None):
            _lib.flute_weights_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def gemm(self, x, y=None, workers: int = 0, stream=None):
        """x: torch f16 [m][k] on cuda -> y f16 [m][n]."""
        import torch
        if x.dtype != torch.float16 or not x.is_cuda or x.dim() != 2 or x.shape[1] != self.k:
            raise InputError(f"x must be a cuda float16 [m][{self.k}] tensor")
        x = x.contiguous()
        m = x.shape[0]
        if y is None:
            y = torch.empty((m, self.n), dtype=torch.float16, device=x.device)
        elif (y.dtype != torch.float16 or y.device != x.device or tuple(y.shape) != (m, self.n)
              or not y.is_contiguous()):
            raise InputError(f"y must be a contiguous float16 [{m}][{self.n}] tensor on {x.device}")
        _check(_lib.flute_gemm(self._h, x.data_ptr(), m, y.data_ptr(), workers,
                               _stream_ptr(stream)))
        return y

    def gemm_peers(self, x, y_ptrs: Sequence[int], ldy: int, ycol0: int, workers: int = 0,
                   stream=None) -> None:
        """Store this GEMM's [m][n] result into every device buffer in y_ptrs
        (row stride ldy, column offset ycol0): the N-sharded all-gather fused
        into the epilogue (flute_gemm_peers)."""
        import torch
        if x.dtype != torch.float16 or not x.is_cuda or x.dim() != 2 or x.shape[1] != self.k:
            raise InputError(f"x must be a cuda float16 [m][{self.k}] tensor")
        x = x.contiguous()
        if not 1 <= len(y_ptrs) <= 8:
            raise ConfigError(f"y_ptrs must hold 1..8 device pointers, got {len(y_ptrs)}")
        if any(int(p) == 0 for p in y_ptrs):
            raise InputError("y_ptrs holds a null device pointer")
        if ycol0 < 0 or ldy < ycol0 + self.n:
            raise ConfigError(f"peer output needs ldy >= ycol0 + n ({ycol0} + {self.n})")
        arr = (C.c_void_p * len(y_ptrs))(*[int(p) for p in y_ptrs])
        _check(_lib.flute_gemm_peers(self._h, x.data_ptr(), x.shape[0], arr, len(y_ptrs), ldy,
                                     ycol0, workers, _stream_ptr(stream)))

    def gemm_host(self, x16: np.ndarray, workers: int = 0, stream=None,
                  out: Optional[np.ndarray] = None) -> np.ndarray:
        """End-to-end: host f16 bits in, host f16 bits out (H2D, GEMM, D2H and a
        stream sync inside).  Pass page-locked arrays (e.g. numpy views of
        pinned torch tensors) for x16/out to make the copies asynchronous DMA."""
        x16 = np.ascontiguousarray(x16, np.uint16)
        m = x16.shape[0]
        if out is None:
            y = np.zeros((m, self.n), np.uint16)
        else:
            if out.dtype != np.uint16 or out.shape != (m, self.n) or not out.flags.c_contiguous:
                raise InputError(f"out must be a C-contiguous uint16 [{m}][{self.n}] array")
            y = out
        _check(_lib.flute_gemm_host(self._h, x16, m, y, workers,
                                    None if stream is None else int(stream)))
        return y


def qgemm(x, w_dev, scales_dev, vlut_dev, bits: int, group: int, n: int, workspace, y=None,
          workers: int = 0, stream=None):
    """Raw device-pointer GEMM (flute_qgemm): all arguments are torch cuda
    tensors in the device layouts."""
    import torch
    m, k = x.shape
    if y is None:
        y = torch.empty((m, n), dtype=torch.float16, device=x.device)
    _check(_lib.flute_qgemm(x.data_ptr(), m, k, n, w_dev.data_ptr(), scales_dev.data_ptr(),
                            vlut_dev.data_ptr(), bits, group, y.data_ptr(), workspace.data_ptr(),
                            workspace.numel() * workspace.element_size(), workers,
                            _stream_ptr(stream)))
    return y


@dataclass
class MatmulResult:
    y: np.ndarray          # f16 bits [m][n]
    stats: dict            # TrafficStats (reference accounting model)


def execute(x16: np.ndarray, slices, k: int, n: int, bits: int, group: int, scales: np.ndarray,
            vlut_words: np.ndarray, dup: int = 1, layout=DEFAULT_LAYOUT, workers: int = 1,
            stages: int = 2, tile_m: int = 0) -> MatmulResult:
    """engine.hpp:72 ``execute(MatmulProblem)`` on the GPU: canonical slices
    (reorder_and_split), [n][k/g] scales and a make_vectorized_lut table, all
    host arrays; returns y (f16 bits) and the reference TrafficStats."""
    x16 = np.ascontiguousarray(x16, np.uint16)
    m = x16.shape[0]
    hi = np.ascontiguousarray(slices[0], np.uint32)
    lo = np.ascontiguousarray(slices[1], np.uint32) if bits == 3 else None
    y = np.zeros((m, n), np.uint16)
    st = np.zeros(7, np.uint64)
    _check(_lib.flute_execute(x16, m, hi, lo.ctypes.data if lo is not None else None, k, n, bits,
                              group, _lay(layout), np.ascontiguousarray(scales, np.uint16),
                              np.ascontiguousarray(vlut_words, np.uint32), dup, workers, stages,
                              tile_m, y, st))
    return MatmulResult(y, dict(zip(TRAFFIC_FIELDS, (int(v) for v in st))))


class HostBatch:
    """A prepared host-buffer batch (flute_host_batch_create): input copies,
    GEMMs and output copies captured once as a CUDA graph; run() replays it
    and returns when every output array is filled.  graph=False keeps the
    eager pipelined path (flute_gemm_host_batch per run).  The host arrays
    are referenced, not copied: refill the inputs in place between runs."""

    def __init__(self, items, workers: int = 0, graph: bool = True):
        cnt = len(items)
        self._args = ((_vp * cnt)(), (C.c_void_p * cnt)(), (C.c_int * cnt)(),
                      (C.c_void_p * cnt)())
        hs, xs, ms, ys = self._args
        self._keep = []
        for i, (dw, x16, out) in enumerate(items):
            if x16.dtype != np.uint16 or x16.ndim != 2 or x16.shape[1] != dw.k \
                    or not x16.flags.c_contiguous:
                raise InputError(f"item {i}: x must be a C-contiguous uint16 [m][{dw.k}] array")
            if (out.dtype != np.uint16 or out.shape != (x16.shape[0], dw.n)
                    or not out.flags.c_contiguous):
                raise InputError(f"item {i}: out must be a C-contiguous uint16 [m][{dw.n}] array")
            self._keep.append((dw, x16, out))
            hs[i] = dw._h
            xs[i] = x16.ctypes.data
            ys[i] = out.ctypes.data
            ms[i] = x16.shape[0]
        self._cnt = cnt
        self._workers = workers
        self._g = None
        if graph:
            g = _vp()
            _check(_lib.flute_host_batch_create(hs, xs, ms, ys, cnt, workers, C.byref(g)))
            self._g = g

    def run(self, stream=None) -> None:
        if self._g is not None:
            _check(_lib.flute_host_batch_run(self._g, _stream_ptr(stream)))
            return
        hs, xs, ms, ys = self._args
        _check(_lib.flute_gemm_host_batch(hs, xs, ms, ys, self._cnt, self._workers,
                                          _stream_ptr(stream)))

    def __del__(self):
        g = getattr(self, "_g", None)
        if g is not None and _lib is not None:
            _lib.flute_host_batch_destroy(g)
            self._g = None


def gemm_host_batch(items, workers: int = 0, stream=None) -> None:
    """End-to-end batch (flute_gemm_host_batch): items = [(DeviceWeights,
    x16 uint16 [m][k] host array, out uint16 [m][n] host array), ...].  Input
    copies, GEMMs and output copies are pipelined; returns when every out is
    filled.  Use page-locked arrays for DMA copies."""
    cnt = len(items)
    hs = (_vp * cnt)()
    xs = (C.c_void_p * cnt)()
    ys = (C.c_void_p * cnt)()
    ms = (C.c_int * cnt)()
    keep = []
    for i, (dw, x16, out) in enumerate(items):
        x16 = np.ascontiguousarray(x16, np.uint16)
        if x16.ndim != 2 or x16.shape[1] != dw.k:
            raise InputError(f"item {i}: x must be uint16 [m][{dw.k}]")
        if (out.dtype != np.uint16 or out.shape != (x16.shape[0], dw.n)
                or not out.flags.c_contiguous):
            raise InputError(f"item {i}: out must be a C-contiguous uint16 [m][{dw.n}] array")
        keep.append(x16)
        hs[i] = dw._h
        xs[i] = x16.ctypes.data
        ys[i] = out.ctypes.data
        ms[i] = x16.shape[0]
    _check(_lib.flute_gemm_host_batch(hs, xs, ms, ys, cnt, workers, _stream_ptr(stream)))


def quantize_matrix_device(w, bits: int, group: int, stream=None):
    """quantize_matrix on the GPU: w torch float32 [k][n] on cuda -> (idx
    uint8 [k][n], scales int16 [n*(k/g)] holding binary16 bits), bit-exact with
    quantize_matrix()."""
    import torch
    if w.dtype != torch.float32 or not w.is_cuda or w.dim() != 2:
        raise InputError("w must be a cuda float32 [k][n] tensor")
    w = w.contiguous()
    k, n = w.shape
    idx = torch.empty((k, n), dtype=torch.uint8, device=w.device)
    sc = torch.empty((n * (k // max(group, 1)),), dtype=torch.int16, device=w.device)
    _check(_lib.flute_quantize_device(w.data_ptr(), k, n, bits, group, idx.data_ptr(),
                                      sc.data_ptr(), _stream_ptr(stream)))
    return idx, sc


def nf_quantiles(bits: int) -> np.ndarray:
    """nf_table.hpp nf_quantiles(bits): raw Phi^-1(p_i), binary64."""
    out = np.zeros(1 << bits, np.float64)
    _check(_lib.flute_nf_quantiles(bits, out))
    return out


def nf_sigma() -> float:
    """nf_table.hpp nf_sigma(): 1 / Phi^-1(1 - delta)."""
    return float(_lib.flute_nf_sigma())


def _calib_pair(w, x_calib):
    w = np.ascontiguousarray(w, np.float32)
    x = np.ascontiguousarray(x_calib, np.float32)
    if w.ndim != 2 or x.ndim != 2:
        raise InputError("w and x_calib must be 2-D")
    if x.shape[1] != w.shape[0]:  # quantize.cpp:145-150
        raise InputError(f"calibration matrix has {x.shape[1]} columns, weights have "
                         f"{w.shape[0]} rows")
    return w, x


def ste_evaluate(w: np.ndarray, x_calib: np.ndarray, bits: int, group: int, sigma_tilde):
    """quantize.hpp ste_evaluate on the GPU: (loss, grad f64 [n*k/g], indices
    u8 [k][n]).  w f32 [k][n], x_calib f32 [m][k], sigma_tilde [n*k/g]."""
    w, x = _calib_pair(w, x_calib)
    k, n = w.shape
    sigma = np.ascontiguousarray(sigma_tilde, np.float64)
    if group > 0 and sigma.size != k // group * n:  # quantize.cpp:155-157
        raise InputError("sigma_tilde has wrong group count")
    loss = C.c_double(0.0)
    grad = np.zeros(sigma.size, np.float64)
    idx = np.zeros((k, n), np.uint8)
    _check(_lib.flute_ste_evaluate(w, x, x.shape[0], k, n, bits, group, sigma, C.byref(loss),
                                   grad, idx))
    return loss.value, grad, idx


def refine_scales(w: np.ndarray, x_calib: np.ndarray, bits: int, group: int, steps: int,
                  lr: float) -> dict:
    """quantize.hpp refine_scales on the GPU: {indices, scales (binary16 bits,
    learned factor folded in), sigma, initial_loss, final_loss}; raises
    OptimizationError (with .step) like the reference."""
    w, x = _calib_pair(w, x_calib)
    k, n = w.shape
    groups = k // max(group, 1) * n
    idx = np.zeros((k, n), np.uint8)
    sc = np.zeros(groups, np.uint16)
    sigma = np.zeros(groups, np.float64)
    losses = np.zeros(2, np.float64)
    step = C.c_int(-1)
    rc = _lib.flute_refine_scales(w, x, x.shape[0], k, n, bits, group, steps, float(lr), idx, sc,
                                  sigma, losses, C.byref(step))
    if rc == OptimizationError.code:
        e = OptimizationError(_lib.flute_last_error().decode())
        e.step = step.value
        raise e
    _check(rc)
    return {"indices": idx, "scales": sc, "sigma": sigma, "initial_loss": float(losses[0]),
            "final_loss": float(losses[1])}


def flte_write(indices: np.ndarray, scales: np.ndarray, table_values: np.ndarray, bits: int,
               group: int, layout=DEFAULT_LAYOUT) -> bytes:
    """Indices + scales + table -> FLTE container bytes (flute_flte_write)."""
    idx = np.ascontiguousarray(indices, np.uint8)
    k, n = idx.shape
    args = (idx, np.ascontiguousarray(scales, np.uint16),
            np.ascontiguousarray(table_values, np.float32), k, n, bits, group, _lay(layout))
    ln = C.c_size_t(0)
    _check(_lib.flute_flte_write(*args, None, 0, C.byref(ln)))
    out = np.zeros(ln.value, np.uint8)
    _check(_lib.flute_flte_write(*args, out.ctypes.data, out.size, C.byref(ln)))
    return out.tobytes()


def flte_info(data: bytes):
    """(bits, group, k, n) of an FLTE container; raises InputError (with the
    reference's section / byte-offset message) on a malformed file."""
    buf = np.frombuffer(bytes(data), np.uint8).copy()
    vals = [C.c_int(0) for _ in range(4)]
    _check(_lib.flute_flte_info(buf, buf.size, *[C.byref(v) for v in vals]))
    return tuple(v.value for v in vals)


@dataclass
class ShardRange:
    n0: int
    n1: int
    w_off: int
    w_bytes: int
    s_off: int
    s_bytes: int


def shard_range(k: int, n: int, bits: int, group: int, world: int, rank: int) -> ShardRange:
    """Columns and device-layout byte ranges owned by `rank` (flute_shard_range)."""
    n0, n1 = C.c_int(0), C.c_int(0)
    v = [C.c_size_t(0) for _ in range(4)]
    _check(_lib.flute_shard_range(k, n, bits, group, world, rank, C.byref(n0), C.byref(n1),
                                  *[C.byref(x) for x in v]))
    return ShardRange(n0.value, n1.value, *[x.value for x in v])


def dequant_all_device(vlut_words: np.ndarray, bits: int, scales: np.ndarray) -> np.ndarray:
    """Run the GEMM kernel's own dequant routine for every pair x scale:
    returns u32 [n_scales][2^(2b)] (reference pair order)."""
    scales = np.ascontiguousarray(scales, np.uint16)
    out = np.zeros((scales.size, 1 << (2 * bits)), np.uint32)
    _check(_lib.flute_dequant_all_device(np.ascontiguousarray(vlut_words, np.uint32), bits, scales,
                                         scales.size, out))
    return out


def mma_fragment(a16: np.ndarray, b16: np.ndarray, c: np.ndarray) -> np.ndarray:
    """mma.hpp:23 on the tensor cores: returns c + a @ b (f16 in, f32 acc)."""
    a16 = np.ascontiguousarray(a16, np.uint16)
    b16 = np.ascontiguousarray(b16, np.uint16)
    c = np.array(c, np.float32, copy=True, order="C")
    m, k = a16.shape
    n = b16.shape[1]
    _check(_lib.flute_mma_fragment(a16, b16, c, m, n, k))
    return c


def debug_times(workers: int, slots: int = 1):
    """Per-CTA ns timeline (diag build, FLUTE_DEBUG_TIMES=slots): for each of
    the ring's `slots` launches, (stamps [workers][16], stage trace
    [workers][64][3])."""
    per = 208 * workers
    out = np.zeros(per * slots, np.uint64)
    _check(_lib.flute_debug_times(out, workers))
    res = [(out[i * per:i * per + 16 * workers].reshape(workers, 16),
            out[i * per + 16 * workers:(i + 1) * per].reshape(workers, 64, 3)) for i in range(slots)]
    return res[0] if slots == 1 else res


def exported_symbols() -> Sequence[str]:
    return tuple(_SIGS)
