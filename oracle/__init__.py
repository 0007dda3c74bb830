"""TEST INFRASTRUCTURE ONLY — ctypes front-end to the CPU oracle.

Two checkers live here, both used solely by ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs:

* :class:`Oracle` — the plain-C restatement (``oracle/flute_oracle.c``) of the
  reference hot path, compiled to ``oracle/_build/liboracle.so``.
* :class:`RefLib` — the *unmodified* reference library (``/root/reference``)
  compiled by ``oracle/Makefile`` into ``oracle/_ref/libflutesim_ref.so`` plus
  the extern-"C" shim ``oracle/ref_shim.cpp``.

The product package (``paper_2407_10960_b200``) never imports this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libflutesim_ref.so")
REF_ROOT = "/root/reference/proj"

DEFAULT_LAYOUT = (16, 64, 64, 16, 8, 16)  # pack.hpp:21-26, cli.cpp:68-69

_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_u16p = np.ctypeslib.ndpointer(np.uint16, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")


class OracleError(RuntimeError):
    def __init__(self, code: int, what: str = ""):
        super().__init__(f"oracle error {code}: {what}")
        self.code = code


def build(ref: bool = True) -> None:
    """Compile the C restatement (always) and the reference .so (when the
    reference sources are present — i.e. in the build container)."""
    subprocess.run(["make", "-s", "-C", HERE, "oracle"], check=True)
    if ref and os.path.isdir(REF_ROOT):
        subprocess.run(["make", "-s", "-C", HERE, "ref"], check=True)


def slice_words(k: int, n: int, w: int) -> int:
    return (k * n * w + 31) // 32


def _lay(layout) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(layout, dtype=np.int32))



class RefineFailed(RuntimeError):
    """OptimizationError of refine_scales (quantize.cpp:246-280), with its step."""

    def __init__(self, step: int, what: str = ""):
        super().__init__(f"refine_scales failed at step {step}: {what}")
        self.step = step


def _ste_call(fn, w, x, bits, group, sigma, chk):
    w = np.ascontiguousarray(w, np.float32)
    x = np.ascontiguousarray(x, np.float32)
    k, n = w.shape
    m = x.shape[0]
    sigma = np.ascontiguousarray(sigma, np.float64)
    loss = C.c_double(0.0)
    grad = np.zeros(sigma.size, np.float64)
    idx = np.zeros((k, n), np.uint8)
    chk(fn(w, x, m, k, n, bits, group, sigma, C.byref(loss), grad, idx), "ste_evaluate")
    return loss.value, grad, idx


def _refine_call(fn, w, x, bits, group, steps, lr, chk, opt_rc, err):
    w = np.ascontiguousarray(w, np.float32)
    x = np.ascontiguousarray(x, np.float32)
    k, n = w.shape
    m = x.shape[0]
    groups = k // group * n
    idx = np.zeros((k, n), np.uint8)
    sc = np.zeros(groups, np.uint16)
    sigma = np.zeros(groups, np.float64)
    losses = np.zeros(2, np.float64)
    step = C.c_int(-1)
    rc = fn(w, x, m, k, n, bits, group, steps, float(lr), idx, sc, sigma, losses, C.byref(step))
    if rc == opt_rc:
        raise RefineFailed(step.value, err())
    chk(rc, "refine_scales")
    return {"indices": idx, "scales": sc, "sigma": sigma, "initial_loss": float(losses[0]),
            "final_loss": float(losses[1])}


class Oracle:
    """The plain-C restatement (flute_oracle.c)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build(ref=False)
        L = self.lib = C.CDLL(path)
        L.orc_f32_to_f16.restype = C.c_uint16
        L.orc_f32_to_f16.argtypes = [C.c_float]
        L.orc_f16_to_f32.restype = C.c_float
        L.orc_f16_to_f32.argtypes = [C.c_uint16]
        L.orc_f16_add.restype = C.c_uint16
        L.orc_f16_add.argtypes = [C.c_uint16, C.c_uint16]
        L.orc_inverse_normal_cdf.restype = C.c_double
        L.orc_inverse_normal_cdf.argtypes = [C.c_double]
        L.orc_nf_table.argtypes = [C.c_int, _f32p]
        L.orc_quantize.argtypes = [_f32p, C.c_int, C.c_int, C.c_int, C.c_int, _u8p, _u16p]
        L.orc_layout_validate.argtypes = [_i32p]
        L.orc_packed_pos.restype = C.c_int64
        L.orc_packed_pos.argtypes = [_i32p, C.c_int, C.c_int, C.c_int, C.c_int]
        L.orc_pack.argtypes = [_u8p, C.c_int, C.c_int, C.c_int, _i32p, _u32p, _u32p]
        L.orc_unpack.argtypes = [C.c_int, C.c_int, C.c_int, _i32p, _u32p, _u32p, _u8p]
        L.orc_vlut.argtypes = [_f32p, C.c_int, C.c_int, _u32p]
        L.orc_vec_dequantize.restype = C.c_uint32
        L.orc_vec_dequantize.argtypes = [C.c_uint32, C.c_uint16]
        L.orc_dequant_table.argtypes = [_u32p, C.c_int, _u16p, C.c_int, _u32p]
        L.orc_plan_stream_k.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, _i64p, C.c_void_p,
                                        C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int64)]
        L.orc_execute.argtypes = [_u16p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _i32p,
                                  _u32p, _u32p, _u16p, _f32p, C.c_int, C.c_int, C.c_int,
                                  _u16p, _u64p]
        L.orc_plan_traffic.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _i32p,
                                       C.c_int, C.c_int, C.c_int, _u64p]
        L.orc_reference_f64.argtypes = [_u16p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                        _u8p, _u16p, _f32p, _f64p]
        L.orc_nf_quantiles.argtypes = [C.c_int, _f64p]
        L.orc_nf_sigma.restype = C.c_double
        L.orc_ste_evaluate.argtypes = [_f32p, _f32p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                       _f64p, C.POINTER(C.c_double), _f64p, _u8p]
        L.orc_refine_scales.argtypes = [_f32p, _f32p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                        C.c_int, C.c_double, _u8p, _u16p, _f64p, _f64p,
                                        C.POINTER(C.c_int)]
        L.orc_reference_f64_mode.argtypes = [_u16p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                             _u8p, _u16p, _f32p, C.c_int, _f64p]

    @staticmethod
    def _chk(rc: int, what: str) -> None:
        if rc != 0:
            raise OracleError(rc, what)

    # -- numerics ---------------------------------------------------------
    def f32_to_f16(self, x: float) -> int:
        return int(self.lib.orc_f32_to_f16(float(x)))

    def f16_to_f32(self, h: int) -> float:
        return float(self.lib.orc_f16_to_f32(int(h)))

    def f16_add(self, a: int, b: int) -> int:
        return int(self.lib.orc_f16_add(a, b))

    # -- producers --------------------------------------------------------
    def nf_table(self, bits: int) -> np.ndarray:
        out = np.zeros(1 << bits, np.float32)
        self._chk(self.lib.orc_nf_table(bits, out), "nf_table")
        return out

    def nf_quantiles(self, bits: int) -> np.ndarray:
        out = np.zeros(1 << bits, np.float64)
        self._chk(self.lib.orc_nf_quantiles(bits, out), "nf_quantiles")
        return out

    def nf_sigma(self) -> float:
        return float(self.lib.orc_nf_sigma())

    def ste_evaluate(self, w, x, bits, group, sigma):
        return _ste_call(self.lib.orc_ste_evaluate, w, x, bits, group, sigma, self._chk)

    def refine_scales(self, w, x, bits, group, steps, lr):
        return _refine_call(self.lib.orc_refine_scales, w, x, bits, group, steps, lr, self._chk, 4,
                            lambda: "loss diverged")

    def quantize(self, w: np.ndarray, bits: int, group: int):
        w = np.ascontiguousarray(w, np.float32)
        k, n = w.shape
        idx = np.zeros((k, n), np.uint8)
        sc = np.zeros(k * n // group, np.uint16)
        self._chk(self.lib.orc_quantize(w, k, n, bits, group, idx, sc), "quantize")
        return idx, sc

    # -- packer -----------------------------------------------------------
    def pack(self, idx: np.ndarray, bits: int, layout=DEFAULT_LAYOUT):
        idx = np.ascontiguousarray(idx, np.uint8)
        k, n = idx.shape
        w0 = 2 if bits == 3 else bits
        s0 = np.zeros(slice_words(k, n, w0), np.uint32)
        s1 = np.zeros(max(1, slice_words(k, n, 1)) if bits == 3 else 1, np.uint32)
        self._chk(self.lib.orc_pack(idx, k, n, bits, _lay(layout), s0, s1), "pack")
        return (s0, s1) if bits == 3 else (s0,)

    def unpack(self, slices, k: int, n: int, bits: int, layout=DEFAULT_LAYOUT) -> np.ndarray:
        s0 = np.ascontiguousarray(slices[0], np.uint32)
        s1 = np.ascontiguousarray(slices[1] if bits == 3 else np.zeros(1, np.uint32), np.uint32)
        out = np.zeros((k, n), np.uint8)
        self._chk(self.lib.orc_unpack(k, n, bits, _lay(layout), s0, s1, out), "unpack")
        return out

    def packed_pos(self, layout, k, n, i, j) -> int:
        return int(self.lib.orc_packed_pos(_lay(layout), k, n, i, j))

    # -- vLUT -------------------------------------------------------------
    def vlut(self, values: np.ndarray, bits: int, dup: int = 1) -> np.ndarray:
        out = np.zeros(1 << (2 * bits), np.uint32)
        self._chk(self.lib.orc_vlut(np.ascontiguousarray(values, np.float32), bits, dup, out),
                  "vlut")
        return out

    def vec_dequantize(self, entry_word: int, scale: int) -> int:
        return int(self.lib.orc_vec_dequantize(entry_word, scale))

    def dequant_table(self, vlut: np.ndarray, bits: int, scales: np.ndarray) -> np.ndarray:
        scales = np.ascontiguousarray(scales, np.uint16)
        out = np.zeros((scales.size, 1 << (2 * bits)), np.uint32)
        self._chk(self.lib.orc_dequant_table(np.ascontiguousarray(vlut, np.uint32), bits, scales,
                                             scales.size, out), "dequant_table")
        return out

    # -- Stream-K ---------------------------------------------------------
    def plan_stream_k(self, tm, tn, tk, workers):
        ranges = np.zeros(2 * workers, np.int64)
        cap = tm * tn
        fx = np.zeros(4 * max(cap, 1), np.int64)
        nf = C.c_int(0)
        slots = C.c_int64(0)
        self._chk(self.lib.orc_plan_stream_k(tm, tn, tk, workers, ranges,
                                             fx.ctypes.data_as(C.c_void_p), cap,
                                             C.byref(nf), C.byref(slots)), "plan_stream_k")
        return ranges.reshape(-1, 2), fx[:4 * nf.value].reshape(-1, 4), slots.value

    # -- engine -----------------------------------------------------------
    def execute(self, x16: np.ndarray, slices, k, n, bits, group, scales, table,
                layout=DEFAULT_LAYOUT, workers=1, stages=2, tile_m=0):
        x16 = np.ascontiguousarray(x16, np.uint16)
        m = x16.shape[0]
        y = np.zeros((m, n), np.uint16)
        st = np.zeros(7, np.uint64)
        s0 = np.ascontiguousarray(slices[0], np.uint32)
        s1 = np.ascontiguousarray(slices[1] if bits == 3 else np.zeros(1, np.uint32), np.uint32)
        self._chk(self.lib.orc_execute(x16, m, k, n, bits, group, _lay(layout), s0, s1,
                                       np.ascontiguousarray(scales, np.uint16),
                                       np.ascontiguousarray(table, np.float32),
                                       workers, stages, tile_m, y, st), "execute")
        return y, st

    def plan_traffic(self, m, k, n, bits, group, layout=DEFAULT_LAYOUT, workers=1, stages=2,
                     tile_m=0):
        st = np.zeros(7, np.uint64)
        self._chk(self.lib.orc_plan_traffic(m, k, n, bits, group, _lay(layout), workers, stages,
                                            tile_m, st), "plan_traffic")
        return st

    def reference_f64(self, x16, idx, bits, group, scales, table, f16_weights=True) -> np.ndarray:
        """binary64 X * W_hat.  f16_weights=True: W_hat = the f16 weights the
        kernel multiplies; False: dequantize_matrix's binary32 weights."""
        x16 = np.ascontiguousarray(x16, np.uint16)
        idx = np.ascontiguousarray(idx, np.uint8)
        m, k = x16.shape
        n = idx.shape[1]
        y = np.zeros((m, n), np.float64)
        self._chk(self.lib.orc_reference_f64_mode(x16, m, k, n, bits, group, idx,
                                                  np.ascontiguousarray(scales, np.uint16),
                                                  np.ascontiguousarray(table, np.float32),
                                                  1 if f16_weights else 0, y),
                  "reference_f64")
        return y


class RefLib:
    """The unmodified reference library (oracle/_ref/libflutesim_ref.so)."""

    @staticmethod
    def available() -> bool:
        return os.path.exists(REF_SO)

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            if os.path.isdir(REF_ROOT):
                build(ref=True)
            else:
                raise FileNotFoundError(f"{path} missing and /root/reference absent")
        L = self.lib = C.CDLL(path, mode=C.RTLD_LOCAL)
        L.fref_last_error.restype = C.c_char_p
        L.fref_f32_to_f16.restype = C.c_uint16
        L.fref_f32_to_f16.argtypes = [C.c_float]
        L.fref_f16_to_f32.restype = C.c_float
        L.fref_f16_to_f32.argtypes = [C.c_uint16]
        L.fref_nf_table.argtypes = [C.c_int, _f32p]
        L.fref_flte_write.argtypes = [_f32p, C.c_int, C.c_int, C.c_int, C.c_int, _i32p, C.c_void_p,
                                      C.c_size_t, C.POINTER(C.c_size_t)]
        L.fref_flte_parse.argtypes = [_u8p, C.c_size_t, C.c_char_p, C.c_size_t,
                                      C.POINTER(C.c_size_t)]
        L.fref_quantize.argtypes = [_f32p, C.c_int, C.c_int, C.c_int, C.c_int, _u8p, _u16p]
        L.fref_pack.argtypes = [_u8p, C.c_int, C.c_int, C.c_int, _i32p, _u32p, _u32p]
        L.fref_unpack.argtypes = [C.c_int, C.c_int, C.c_int, _i32p, _u32p, _u32p, _u8p]
        L.fref_packed_pos.restype = C.c_longlong
        L.fref_packed_pos.argtypes = [_i32p, C.c_int, C.c_int, C.c_int, C.c_int]
        L.fref_vlut.argtypes = [_f32p, C.c_int, C.c_int, _u32p]
        L.fref_vec_dequantize.argtypes = [_f32p, C.c_int, C.c_uint32, C.c_uint16,
                                          C.POINTER(C.c_uint32)]
        L.fref_plan_stream_k.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, _i64p, C.c_void_p,
                                         C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_longlong)]
        L.fref_execute.argtypes = [_u16p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _i32p,
                                   _u32p, _u32p, _u16p, _f32p, C.c_int, C.c_int, C.c_int,
                                   C.c_int, C.c_int, _u16p, _u64p]
        L.fref_ste_evaluate.argtypes = [_f32p, _f32p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                        _f64p, C.POINTER(C.c_double), _f64p, _u8p]
        L.fref_refine_scales.argtypes = [_f32p, _f32p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                         C.c_int, C.c_double, _u8p, _u16p, _f64p, _f64p,
                                         C.POINTER(C.c_int)]
        L.fref_plan_traffic.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _i32p,
                                        C.c_int, C.c_int, C.c_int, C.c_int, _u64p]

    def _chk(self, rc: int, what: str) -> None:
        if rc != 0:
            raise OracleError(rc, f"{what}: {self.lib.fref_last_error().decode()}")

    def f32_to_f16(self, x: float) -> int:
        return int(self.lib.fref_f32_to_f16(float(x)))

    def flte_write(self, w: np.ndarray, bits: int, group: int, layout=DEFAULT_LAYOUT) -> bytes:
        """quantize_matrix + reorder_and_split + write_flte of the reference."""
        w = np.ascontiguousarray(w, np.float32)
        k, n = w.shape
        ln = C.c_size_t(0)
        lay = _lay(layout)
        rc = self.lib.fref_flte_write(w, k, n, bits, group, lay, None, 0, C.byref(ln))
        if rc:
            raise OracleError(rc, self.lib.fref_last_error().decode())
        out = np.zeros(ln.value, np.uint8)
        rc = self.lib.fref_flte_write(w, k, n, bits, group, lay, out.ctypes.data, out.size,
                                      C.byref(ln))
        if rc:
            raise OracleError(rc, self.lib.fref_last_error().decode())
        return out.tobytes()

    def flte_parse(self, data: bytes):
        """None if the reference's read_flte accepts data, else (section, offset)."""
        buf = np.frombuffer(bytes(data), np.uint8).copy()
        sec = C.create_string_buffer(64)
        off = C.c_size_t(0)
        rc = self.lib.fref_flte_parse(buf, buf.size, sec, 64, C.byref(off))
        if rc == 0:
            return None
        if rc == 5:
            return sec.value.decode(), off.value
        raise OracleError(rc, self.lib.fref_last_error().decode())

    def nf_table(self, bits: int) -> np.ndarray:
        out = np.zeros(1 << bits, np.float32)
        self._chk(self.lib.fref_nf_table(bits, out), "nf_table")
        return out

    def ste_evaluate(self, w, x, bits, group, sigma):
        return _ste_call(self.lib.fref_ste_evaluate, w, x, bits, group, sigma, self._chk)

    def refine_scales(self, w, x, bits, group, steps, lr):
        return _refine_call(self.lib.fref_refine_scales, w, x, bits, group, steps, lr, self._chk, 5,
                            lambda: self.lib.fref_last_error().decode())

    def quantize(self, w: np.ndarray, bits: int, group: int):
        w = np.ascontiguousarray(w, np.float32)
        k, n = w.shape
        idx = np.zeros((k, n), np.uint8)
        sc = np.zeros(k * n // group, np.uint16)
        self._chk(self.lib.fref_quantize(w, k, n, bits, group, idx, sc), "quantize")
        return idx, sc

    def pack(self, idx: np.ndarray, bits: int, layout=DEFAULT_LAYOUT):
        idx = np.ascontiguousarray(idx, np.uint8)
        k, n = idx.shape
        w0 = 2 if bits == 3 else bits
        s0 = np.zeros(slice_words(k, n, w0), np.uint32)
        s1 = np.zeros(max(1, slice_words(k, n, 1)) if bits == 3 else 1, np.uint32)
        self._chk(self.lib.fref_pack(idx, k, n, bits, _lay(layout), s0, s1), "pack")
        return (s0, s1) if bits == 3 else (s0,)

    def unpack(self, slices, k, n, bits, layout=DEFAULT_LAYOUT):
        s0 = np.ascontiguousarray(slices[0], np.uint32)
        s1 = np.ascontiguousarray(slices[1] if bits == 3 else np.zeros(1, np.uint32), np.uint32)
        out = np.zeros((k, n), np.uint8)
        self._chk(self.lib.fref_unpack(k, n, bits, _lay(layout), s0, s1, out), "unpack")
        return out

    def vlut(self, values, bits, dup=1):
        out = np.zeros(1 << (2 * bits), np.uint32)
        self._chk(self.lib.fref_vlut(np.ascontiguousarray(values, np.float32), bits, dup, out),
                  "vlut")
        return out

    def vec_dequantize(self, values, bits, pair, scale) -> int:
        o = C.c_uint32(0)
        self._chk(self.lib.fref_vec_dequantize(np.ascontiguousarray(values, np.float32), bits,
                                               pair, scale, C.byref(o)), "vec_dequantize")
        return o.value

    def plan_stream_k(self, tm, tn, tk, workers):
        ranges = np.zeros(2 * workers, np.int64)
        cap = tm * tn
        fx = np.zeros(4 * max(cap, 1), np.int64)
        nf = C.c_int(0)
        slots = C.c_longlong(0)
        self._chk(self.lib.fref_plan_stream_k(tm, tn, tk, workers, ranges,
                                              fx.ctypes.data_as(C.c_void_p), cap, C.byref(nf),
                                              C.byref(slots)), "plan_stream_k")
        return ranges.reshape(-1, 2), fx[:4 * nf.value].reshape(-1, 4), slots.value

    def execute(self, x16, slices, k, n, bits, group, scales, table, layout=DEFAULT_LAYOUT,
                workers=1, stages=2, tile_m=0, dup=1, parallel=True):
        x16 = np.ascontiguousarray(x16, np.uint16)
        m = x16.shape[0]
        y = np.zeros((m, n), np.uint16)
        st = np.zeros(7, np.uint64)
        s0 = np.ascontiguousarray(slices[0], np.uint32)
        s1 = np.ascontiguousarray(slices[1] if bits == 3 else np.zeros(1, np.uint32), np.uint32)
        self._chk(self.lib.fref_execute(x16, m, k, n, bits, group, _lay(layout), s0, s1,
                                        np.ascontiguousarray(scales, np.uint16),
                                        np.ascontiguousarray(table, np.float32), dup, workers,
                                        stages, tile_m, 1 if parallel else 0, y, st), "execute")
        return y, st

    def plan_traffic(self, m, k, n, bits, group, layout=DEFAULT_LAYOUT, workers=1, stages=2,
                     dup=1, tile_m=0):
        st = np.zeros(7, np.uint64)
        self._chk(self.lib.fref_plan_traffic(m, k, n, bits, group, _lay(layout), workers, stages,
                                             dup, tile_m, st), "plan_traffic")
        return st
