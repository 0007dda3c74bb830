// flute-b200 — register-level LUT dequantization (FLUTE §3.2, Alg. 1 "vectorized
// lookup"; reference semantics vec_lut.cpp:39-48).
//
// Shared-memory vLUT: entry e occupies one 256-byte row; lane l reads its own
// copy at e*256 + 4l, so a warp's 32 lookups always hit 32 distinct banks
// (duplication 32, conflict-free).  The byte offset e*256 + 4l is produced by a
// single PRMT from a byte vector of device pair indices (byte p -> bits 8..15,
// lane*4 -> bits 0..7), which ptxas folds into LDS [R + UR + imm].
//
// Dequant: half2 = vLUT[e] * (s, s) with one HMUL2 (mul.rn.f16x2).  The product
// of two binary16 values is exact in binary32, so f16(f32(s) * f32(T)) — the
// reference rule — equals the RNE f16x2 product bit for bit (subnormals are
// kept by f16 arithmetic on sm_100).
//
// Per lane and 16-deep k step, the device layout (host_pack.cpp) gives 16 pair
// indices q = 4j + p (atom j = 16-column block, p = A-fragment register):
//   4-bit: uint4, byte p of word j = pair 4j+p                      (8 bits/pair)
//   2-bit: uint2, word h: low nibbles of bytes 0..3 = pairs 8h+0..3, high
//          nibbles = pairs 8h+4..7                                   (4 bits/pair)
//   3-bit: three u32 words A, B, C (uint2 hi = {A, B}, u32 lo = C).  The
//          6-bit device index of pair 4j+p is (hi_k<<2|hi_k1)<<2 | (lo_k<<1|
//          lo_k1) (the 2+1-bit plane split, FLUTE §3.1).  For atoms j = 0, 1,
//          2 it sits in bits 0..5 of byte p of word A, B, C; atom 3's index is
//          spread over bits 6..7 of byte p of A (index bits 0-1), B (2-3) and
//          C (4-5).  Atoms 0-2 need no instruction at all, atom 3 two shifts
//          folded into two LOP3s; bits 6..7 of every index byte are left as
//          garbage, which the 256-entry table (64 entries replicated four
//          times) ignores.
#pragma once

#include "ptx.cuh"

namespace flute_dev {

inline constexpr int kLutRowBytes = 256;

// Rows of the shared-memory table: 256 for every bit width — the 2^(2b)
// entries replicated 256 / 2^(2b) times, so index bytes may carry don't-care
// high bits (atom_index_bytes<2>, <3>) and need no masking.
template <int BITS>
inline constexpr int kTableRows = 256;

// (m & a) | (~m & b), one LOP3
__device__ __forceinline__ uint32_t bitselect(uint32_t m, uint32_t a, uint32_t b) {
  return (m & a) | (~m & b);
}

template <int BITS>
struct LaneBits;
template <>
struct LaneBits<4> {
  uint4 w;
};
template <>
struct LaneBits<2> {
  uint2 w;
};
template <>
struct LaneBits<3> {
  uint2 hi;
  uint32_t lo;
};

// Byte vector of the 4 device pair indices of atom j (byte p = register p).
template <int BITS>
__device__ __forceinline__ uint32_t atom_index_bytes(const LaneBits<BITS>& lb, int j);

template <>
__device__ __forceinline__ uint32_t atom_index_bytes<4>(const LaneBits<4>& lb, int j) {
  return j == 0 ? lb.w.x : j == 1 ? lb.w.y : j == 2 ? lb.w.z : lb.w.w;
}
// (bits 4..7 of each byte undefined: index a 256-row table, or mask)
template <>
__device__ __forceinline__ uint32_t atom_index_bytes<2>(const LaneBits<2>& lb, int j) {
  const uint32_t w = (j >> 1) ? lb.w.y : lb.w.x;
  return (j & 1) ? w >> 4 : w;
}
// (bits 6..7 of each byte undefined: index a 256-entry table, or mask)
template <>
__device__ __forceinline__ uint32_t atom_index_bytes<3>(const LaneBits<3>& lb, int j) {
  if (j == 0) return lb.hi.x;
  if (j == 1) return lb.hi.y;
  if (j == 2) return lb.lo;
  // bits 0-1 from A >> 6, bits 2-3 from B >> 4, bits 4-5 from C >> 2
  const uint32_t ab = bitselect(0x03030303u, lb.hi.x >> 6, lb.hi.y >> 4);
  return bitselect(0x0F0F0F0Fu, ab, lb.lo >> 2);
}

// Inverse of atom_index_bytes<3>: the three lane words of 16 six-bit device
// indices d[4j + p] (the packers' and the self-check's encoder).
__host__ __device__ inline void pack_lane_w3(const uint32_t (&d)[16], uint32_t& a, uint32_t& b,
                                             uint32_t& c) {
  a = b = c = 0u;
  for (int p = 0; p < 4; ++p) {
    const uint32_t d3 = d[12 + p];
    a |= (d[p] | (d3 & 3u) << 6) << (8 * p);
    b |= (d[4 + p] | ((d3 >> 2) & 3u) << 6) << (8 * p);
    c |= (d[8 + p] | ((d3 >> 4) & 3u) << 6) << (8 * p);
  }
}

// The four A-fragment registers of atom j: a[p] = vLUT[idx_p] * (s, s), with
// regs 0/2 (column g) scaled by the low half of `scales` and regs 1/3 (column
// g+8) by the high half.  The half broadcast folds into the HMUL2 operand
// selector (.H0_H0 / .H1_H1), so it costs no instruction.
__device__ __forceinline__ void lut_dequant4(uint32_t idx_bytes, uint32_t lane4, uint32_t lut_base,
                                             uint32_t scales, uint32_t (&a)[4]) {
  const __half2 s2 = *reinterpret_cast<const __half2*>(&scales);
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    const uint32_t off = prmt(idx_bytes, lane4, 0x5504u | (static_cast<uint32_t>(p) << 4));
    uint32_t v = lds32_const(lut_base + off);
    const __half2 r = __hmul2(*reinterpret_cast<const __half2*>(&v),
                              (p & 1) ? __high2half2(s2) : __low2half2(s2));
    a[p] = *reinterpret_cast<const uint32_t*>(&r);
  }
}

// Compact-table variant (128-byte rows: the 32 lane copies only, no partial-
// sum rows in the gaps): one PRMT puts idx << 8 | lane*8 together and a shift
// halves it to idx * 128 + lane * 4.
__device__ __forceinline__ void lut_dequant4_r128(uint32_t idx_bytes, uint32_t lane8, uint32_t lut_base,
                                                  uint32_t scales, uint32_t (&a)[4]) {
  const __half2 s2 = *reinterpret_cast<const __half2*>(&scales);
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    const uint32_t off = prmt(idx_bytes, lane8, 0x5504u | (static_cast<uint32_t>(p) << 4)) >> 1;
    uint32_t v = lds32_const(lut_base + off);
    const __half2 r = __hmul2(*reinterpret_cast<const __half2*>(&v),
                              (p & 1) ? __high2half2(s2) : __low2half2(s2));
    a[p] = *reinterpret_cast<const uint32_t*>(&r);
  }
}
template <int BITS, int NTHREADS>
__device__ __forceinline__ void fill_lut_r128(uint32_t lut_base, const uint32_t* __restrict__ vlut, int tid) {
  constexpr int kEntries = kTableRows<BITS>;
  constexpr int kSrcMask = (1 << (2 * BITS)) - 1;
  constexpr int kChunks = kEntries * 8;  // 8 x 16-byte chunks = the 32 lane copies
  constexpr int kPer = (kChunks + NTHREADS - 1) / NTHREADS;
  uint32_t v[kPer];
#pragma unroll
  for (int i = 0; i < kPer; ++i) {
    const int c = tid + i * NTHREADS;
    v[i] = c < kChunks ? __ldg(vlut + ((c >> 3) & kSrcMask)) : 0u;
  }
#pragma unroll
  for (int i = 0; i < kPer; ++i) {
    const int c = tid + i * NTHREADS;
    if (c < kChunks) sts128(lut_base + (c >> 3) * 128 + (c & 7) * 16, make_uint4(v[i], v[i], v[i], v[i]));
  }
}

// The two halves of lut_dequant4, for callers that batch the lookups of
// several atoms ahead of their MMAs (more loads in flight per warp).
__device__ __forceinline__ void lut_lookup4(uint32_t idx_bytes, uint32_t lane4, uint32_t lut_base,
                                            uint32_t (&v)[4]) {
#pragma unroll
  for (int p = 0; p < 4; ++p)
    v[p] = lds32_const(lut_base + prmt(idx_bytes, lane4, 0x5504u | (static_cast<uint32_t>(p) << 4)));
}
__device__ __forceinline__ void lut_scale4(const uint32_t (&v)[4], uint32_t scales, uint32_t (&a)[4]) {
  const __half2 s2 = *reinterpret_cast<const __half2*>(&scales);
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    const __half2 r = __hmul2(*reinterpret_cast<const __half2*>(&v[p]),
                              (p & 1) ? __high2half2(s2) : __low2half2(s2));
    a[p] = *reinterpret_cast<const uint32_t*>(&r);
  }
}

// Expand the 2^(2b) device-order vLUT words into the 32-copy shared table.
// Called by `nthreads` threads with ids [0, nthreads).
template <int BITS, int NTHREADS, int ROWS = kTableRows<BITS>>
__device__ __forceinline__ void fill_lut(uint32_t lut_base, const uint32_t* __restrict__ vlut,
                                         int tid) {
  constexpr int kEntries = ROWS;
  constexpr int kSrcMask = (1 << (2 * BITS)) - 1;
  constexpr int kChunks = kEntries * 8;  // 8 x 16-byte chunks = the 32 lane copies
  constexpr int kPer = (kChunks + NTHREADS - 1) / NTHREADS;
  // All global loads first (one latency), then the shared stores.
  uint32_t v[kPer];
#pragma unroll
  for (int i = 0; i < kPer; ++i) {
    const int c = tid + i * NTHREADS;
    v[i] = c < kChunks ? __ldg(vlut + ((c >> 3) & kSrcMask)) : 0u;
  }
#pragma unroll
  for (int i = 0; i < kPer; ++i) {
    const int c = tid + i * NTHREADS;
    if (c < kChunks) sts128(lut_base + (c >> 3) * kLutRowBytes + (c & 7) * 16,
                            make_uint4(v[i], v[i], v[i], v[i]));
  }
}

// Broadcast the halves of a packed scale word: (lo, lo) and (hi, hi).
__device__ __forceinline__ uint32_t dup_lo(uint32_t s) { return prmt(s, s, 0x1010u); }
__device__ __forceinline__ uint32_t dup_hi(uint32_t s) { return prmt(s, s, 0x3232u); }

}  // namespace flute_dev
