// flute-b200 — the LUT-dequant GEMM for the compute-bound regime (M >= 64) on
// the 5th-generation tensor cores (tcgen05 / TMEM), sm_100a.
//
// Same device layout, vLUT and scale blocks as the memory-bound kernel
// (qgemm_kernel.cuh), so one DeviceWeights upload serves every M.
//
// CTA tile: 128 output columns (two 64-column units, UMMA M = 128 with W^T as
// the A operand) x BN rows of X (UMMA N = BN), full or split K.  Roles:
//  * TMA warp (8): per 128-deep stage, one bulk copy of the two units' packed
//    weights (contiguous), one of their group scales, and two 128B-swizzled
//    TMA boxes {64 k, BN rows} of X — the canonical K-major SW128 UMMA layout.
//  * 8 dequant warps (0..7): warp w dequantises k-step w of both units through
//    the 32-way duplicated smem vLUT (PRMT -> LDS -> HMUL2, bit-identical to
//    vec_dequantize) and stores the f16 pairs into the A tile in the same
//    K-major SW128 layout (row n at n*128 B within 1024 B atoms, 16-byte chunk
//    index XOR (n & 7)), then fence.proxy.async and arrive.
//  * MMA warp (9): one elected thread issues 8 tcgen05.mma.kind::f16 per stage
//    (2 swizzle atoms x 4 K=16 steps) into the fp32 TMEM accumulator
//    (128 lanes x BN columns) and commits to the stage's empty barrier.
//  * Epilogue (warps 0..3 after their last stage): tcgen05.ld 32x32b.x16 of
//    their 32 TMEM lanes (= 32 output columns), f16 round, store Y[m][n]
//    (or the fp32 split-K partial, reduced in fixed split order by a second
//    kernel).
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <string>
#include <type_traits>

#include "dequant.cuh"
#include "device_api.h"
#include "flutesim/errors.hpp"
#include "ptx.cuh"

namespace flute_dev {

namespace tc {

// 16 dequant warps in four groups of 4 taking 64-k stages round-robin (the
// per-stage dequant is a latency chain — packed/scale loads, vLUT lookups,
// tcgen05.st, wait::st — so four stages are in flight per SM), then the
// producers and the MMA issuer.
constexpr int kDqWarps = 16;
constexpr int kGroupWarps = 4;
constexpr int kGroups = kDqWarps / kGroupWarps;
constexpr int kWWarp = 16;  // weights + scales producer
constexpr int kXWarp = 17;  // X producer
// MMA issuers: warp kMmaWarp + j takes stages i with i % kNumAcc<BN> == j and
// accumulates into its own TMEM accumulator (columns [j*BN, (j+1)*BN)); the
// epilogue adds the accumulators in j order.  One thread's tcgen05.mma issue
// costs ~80-120 cycles whatever N is (tools/umma_chain.cu), so below N = 256
// a single issuer cannot keep the tensor pipe busy; 2 issuers saturate it at
// N = 128, 4 at N = 64.
constexpr int kMmaWarp = 18;
template <int BN>
constexpr int kNumAcc = BN >= 256 ? 1 : BN >= 128 ? 2 : 4;  // = MMA issuer warps
constexpr int threads_for_bn(int bn) { return 32 * (18 + (bn >= 256 ? 1 : bn >= 128 ? 2 : 4)); }
constexpr int kUnitK = 128;
constexpr int kMaxW = 8, kMaxA = 8, kMaxX = 8;
// The dequantised A tiles live in tensor memory ("TS" MMA): the accumulator
// takes columns [0, BN), A slot s columns [kAcol + 32 s, +32) (128 lanes = the
// 128 output columns n, 32 columns = 64 k as f16 pairs).
constexpr int kTmemCols = 512;
constexpr int kAcol = 256;
// A W-ring slot holds kWK whole units (128 k each) of both n-tiles: one bulk
// copy of weights and one of scales per n-tile and slot (few, large copies).
constexpr int kWK = 2;

struct Params {
  const uint8_t* w;
  const uint8_t* sc;
  const uint32_t* vlut;
  __half* y;
  float* part;  // split-K partials [split][m][n] (splits > 1)
  int m, n;
  int tiles_k;   // 128-deep units per column
  int tiles_n;   // 64-column tiles
  int gp;        // padded groups per column
  int group_shift;
  int splits;
  int sw, sx, sa;  // W / X / A ring depths
  int ngw;       // scale groups of one n-tile in a W slot (kWK units, + 1 for an unaligned start)
  uint32_t bar_off, x_off, w_off, w_stage;
  unsigned long long* trace;  // diag build, FLUTE_TC_TRACE: [cta][4] + [cta][64 stages][8] (ns)
  int diag;                   // diag build, FLUTE_TC_DIAG bits: 1 skip tcgen05.st, 2 skip the MMAs
};

__device__ __forceinline__ unsigned long long tc_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#ifdef FLUTE_DIAGNOSTICS
#define TC_TRACE(slot, v)                                                                     \
  do {                                                                                        \
    if (p.trace) p.trace[(blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z)) * 4 + (slot)] = (v); \
  } while (0)
#define TC_STAGE(i, slot)                                                                      \
  do {                                                                                         \
    if (p.trace && (i) < 64)                                                                   \
      p.trace[static_cast<size_t>(gridDim.x * gridDim.y * gridDim.z) * 4 +                     \
              ((blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z)) * 64 + (i)) * 8 + (slot)] = tc_now(); \
  } while (0)
#else
#define TC_TRACE(slot, v) \
  do {                    \
  } while (0)
#define TC_STAGE(i, slot) \
  do {                    \
  } while (0)
#endif

__device__ __forceinline__ uint64_t smem_desc_sw128(uint32_t addr) {
  // K-major, 128B swizzle: start >> 4, LBO = 1 (unused for swizzled K-major),
  // SBO = 1024 B (8 rows x 128 B), version 1 (sm100), layout SWIZZLE_128B = 2.
  return static_cast<uint64_t>((addr >> 4) & 0x3FFFu) | (static_cast<uint64_t>(1) << 16) |
         (static_cast<uint64_t>(1024 >> 4) << 32) | (static_cast<uint64_t>(1) << 46) |
         (static_cast<uint64_t>(2) << 61);
}

template <int BN>
constexpr uint32_t instr_desc() {
  // kind::f16: D f32 (bits 4-5 = 1), A/B f16 (0), K-major both, N >> 3 at 17,
  // M >> 4 at 24 (M = 128).
  return (1u << 4) | (static_cast<uint32_t>(BN >> 3) << 17) | (static_cast<uint32_t>(128 >> 4) << 24);
}

// A from tensor memory (address = column base of the K = 16 slice), B = X^T
// from shared memory (descriptor), D in tensor memory.
__device__ __forceinline__ void umma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                        uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// 16 lanes x 8 columns from the mma.sync A-fragment registers of one 16 x 16
// atom: lane L <- (row g = L, pair t) / (row g + 8, pair t) in r0 / r1,
// pairs t + 4 in r2 / r3 (the fragment order IS the 16x128b pattern)
__device__ __forceinline__ void tmem_st_atom(uint32_t taddr, const uint32_t (&a)[4]) {
  asm volatile("tcgen05.st.sync.aligned.16x128b.x2.b32 [%0], {%1, %2, %3, %4};" ::"r"(taddr), "r"(a[0]),
               "r"(a[1]), "r"(a[2]), "r"(a[3])
               : "memory");
}
__device__ __forceinline__ void umma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
               : "memory");
}

// Ring position of item i in a ring of `depth` slots.
struct Slot {
  int s;
  uint32_t ph;
  __device__ __forceinline__ Slot(int i, int depth) : s(i % depth), ph(static_cast<uint32_t>(i / depth) & 1u) {}
};

// Stages are 64 k deep (one 128B-swizzle atom of the A and X tiles): stage i
// covers k [kt*128 + 64*h, +64) with kt = kt_lo + i/2, h = i & 1.  Three
// independent rings so each resource runs as far ahead as its size allows:
//  * W ring (sw slots): the two units' packed weights for the stage + their
//    group scales, filled by the W warp (the first sw stages before the
//    programmatic-dependent-launch wait — weights do not depend on the
//    previous kernel); freed by every dequant lane once read;
//  * A ring (2 slots): the dequantised W^T tile [128 n][64 k] f16, K-major
//    SW128, written by the 8 dequant warps; freed by the MMA commit;
//  * X ring (sx slots): the X tile [BN rows][64 k] (one TMA box, the
//    canonical K-major SW128 UMMA layout), filled by the X warp after the
//    PDL wait; freed by the MMA commit.
template <int BITS, int BN>
__global__ void __launch_bounds__(threads_for_bn(BN), 1)
    qgemm_tc_kernel(const __grid_constant__ CUtensorMap tmap_x, const Params p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  constexpr int kSubBytes = BITS * 1024;      // one unit's packed weights (128 k)
  constexpr int kSlotW = kWK * kSubBytes;      // one n-tile's weights in a W slot
  constexpr uint32_t kXBytes = BN * 128;       // [BN rows][64 k] f16

  const uint32_t base = smem_u32(smem);
  const uint32_t lut = base;
  const uint32_t bars = base + p.bar_off;
  auto w_full = [&](int s) { return bars + 8 * s; };
  auto w_empty = [&](int s) { return bars + 8 * (kMaxW + s); };
  auto a_full = [&](int s) { return bars + 8 * (2 * kMaxW + s); };
  auto a_empty = [&](int s) { return bars + 8 * (2 * kMaxW + kMaxA + s); };
  auto x_full = [&](int s) { return bars + 8 * (2 * kMaxW + 2 * kMaxA + s); };
  auto x_empty = [&](int s) { return bars + 8 * (2 * kMaxW + 2 * kMaxA + kMaxX + s); };
  const uint32_t acc_full = bars + 8 * (2 * kMaxW + 2 * kMaxA + 2 * kMaxX);
  const uint32_t tmem_slot = acc_full + 8;  // tcgen05.alloc writes the TMEM base here
  auto x_at = [&](int s) { return base + p.x_off + s * kXBytes; };
  auto w_at = [&](int s) { return base + p.w_off + s * p.w_stage; };

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int pair = blockIdx.x;  // 128-column tile = units' n-tiles 2*pair, 2*pair+1
  const int m0 = blockIdx.y * BN;
  const int z = blockIdx.z;
  const int kt_lo = z * p.tiles_k / p.splits;
  const int kt_hi = (z + 1) * p.tiles_k / p.splits;
  const int nk = (kt_hi - kt_lo) * 2;  // 64-deep stages
  const int nt0 = 2 * pair;
  const bool has_u1 = nt0 + 1 < p.tiles_n;
  const int SW = p.sw, SX = p.sx, SA = p.sa;
  if (threadIdx.x == 0) TC_TRACE(0, tc_now());

  if (threadIdx.x == 0) {
    for (int s = 0; s < SW; ++s) {
      mbar_init(w_full(s), 1);
      mbar_init(w_empty(s), kDqWarps * 32);
    }
    for (int s = 0; s < SA; ++s) {
      mbar_init(a_full(s), kGroupWarps * 32);  // the stage's group
      mbar_init(a_empty(s), 1);
    }
    for (int s = 0; s < SX; ++s) {
      mbar_init(x_full(s), 1);
      mbar_init(x_empty(s), 1);
    }
    mbar_init(acc_full, kNumAcc<BN>);  // one commit per MMA issuer warp
    fence_mbar_init();
  }
  if (warp == kMmaWarp) {
    // TMEM: the fp32 accumulator (BN columns) + the A ring (one CTA per SM)
    tmem_alloc(tmem_slot, kTmemCols);
  }
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(smem + (tmem_slot - base));
  pdl_launch_dependents();

  if (warp == kWWarp) {
    // ===================== weights + scales producer =====================
    if (elect_one()) {
      const uint64_t pol = policy_evict_first();
      const int units_pair = has_u1 ? 2 : 1;
      const int nw = (kt_hi - kt_lo + kWK - 1) / kWK;  // W slots
      for (int j = 0; j < nw; ++j) {
        const Slot ws(j, SW);
        if (j >= SW) mbar_wait_sleep(w_empty(ws.s), ws.ph ^ 1u);
        const int kt0 = kt_lo + j * kWK;
        const int nu = kt_hi - kt0 < kWK ? kt_hi - kt0 : kWK;
        const int glo = (kt0 * kUnitK) >> p.group_shift;
        const int ng = ((((kt0 + nu) * kUnitK) - 1) >> p.group_shift) - glo + 1;
        const uint32_t st = w_at(ws.s);
        mbar_arrive_expect_tx(w_full(ws.s), units_pair * (nu * kSubBytes + ng * 128));
        for (int u = 0; u < units_pair; ++u) {
          const size_t unit = static_cast<size_t>(nt0 + u) * p.tiles_k + kt0;
          bulk_g2s_hint(st + u * kSlotW, p.w + unit * kSubBytes, nu * kSubBytes, w_full(ws.s), pol);
          bulk_g2s(st + 2 * kSlotW + u * p.ngw * 128, p.sc + (static_cast<size_t>(nt0 + u) * p.gp + glo) * 128,
                   ng * 128, w_full(ws.s));
        }
      }
    }
  } else if (warp == kXWarp) {
    // ===================== X producer =====================
    if (elect_one()) {
      prefetch_tmap(&tmap_x);
      pdl_wait();  // X belongs to the previous kernel in the stream
      TC_TRACE(3, tc_now());
      for (int i = 0; i < nk; ++i) {
        const Slot xs(i, SX);
        // (one "slot empty" barrier per A / X slot pair: one commit per stage)
        // X slot xs.s is free once the MMAs of stage i - SX have completed:
        // BN < 256 (several MMA issuers, stages retire out of order) — their
        // own X-release commit; BN = 256 (one issuer, SX == SA) — the A-ring
        // release of that stage (a second commit per stage costs the single
        // issuer ~4 % there)
        if (i >= SX) {
          if constexpr (BN < 256) {
            mbar_wait_sleep(x_empty(xs.s), xs.ph ^ 1u);
          } else {
            const Slot prev(i - SX, SA);
            mbar_wait_sleep(a_empty(prev.s), prev.ph);
          }
        }
        const int kt = kt_lo + (i >> 1), h = i & 1;
        mbar_arrive_expect_tx(x_full(xs.s), kXBytes);
        tma_2d_g2s(x_at(xs.s), &tmap_x, kt * kUnitK + 64 * h, m0, x_full(xs.s));
      }
    }
  } else if (warp >= kMmaWarp) {
    // ===================== MMA issuers =====================
    constexpr uint32_t idesc = instr_desc<BN>();
    constexpr int NA = kNumAcc<BN>;
    const int ja = warp - kMmaWarp;  // this issuer's accumulator
    const uint32_t dacc = tmem + static_cast<uint32_t>(ja * BN);
    for (int i = ja; ja < NA && i < nk; i += NA) {
      const Slot as(i, SA), xs(i, SX);
      mbar_wait(a_full(as.s), as.ph);
      if (lane == 0) TC_STAGE(i, 7);
      mbar_wait(x_full(xs.s), xs.ph);
      if (lane == 0) TC_STAGE(i, 3);
      tmem_fence_after();
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const uint64_t bd = smem_desc_sw128(x_at(xs.s) + kk * 32);
#ifdef FLUTE_DIAGNOSTICS
          if (p.diag & 2) continue;
#endif
          umma_ts(dacc, tmem + kAcol + 32 * as.s + 8 * kk, bd, idesc, (i >= NA || kk) ? 1u : 0u);
        }
        umma_commit(a_empty(as.s));  // this stage's A (and, BN = 256, X) slot free once read
        if constexpr (BN < 256) umma_commit(x_empty(xs.s));
      }
      __syncwarp();
    }
    // every issuer arrives once (an issuer without stages arrives at once)
    if (elect_one()) umma_commit(acc_full);
    __syncwarp();
  } else {
    // ===================== dequant warps (0..15) =====================
    fill_lut_r128<BITS, kDqWarps * 32>(lut, p.vlut, threadIdx.x);
    named_bar_sync(1, kDqWarps * 32);
    const uint32_t lane8 = static_cast<uint32_t>(lane) * 8u;
    // group grp = warp >> 2 takes stages i with i % 4 == grp.  Its warp owns
    // TMEM subpartition sp = warp & 3 (the 32 output columns 32 sp .. 32 sp +
    // 31 = unit sp >> 1, atoms 2 (sp & 1) and 2 (sp & 1) + 1) for all four
    // k-steps of the stage.
    const int grp = warp >> 2;
    const int sp = warp & 3;
    const int u = sp >> 1;
    const int jb = 2 * (sp & 1);  // first atom of this warp
    const uint32_t s_lane = (lane >> 2) * 16;
    const bool active = u == 0 || has_u1;
    const uint32_t t_lane = tmem + (static_cast<uint32_t>(32 * sp) << 16) + kAcol;
    for (int i = grp; i < nk; i += kGroups) {
      const int j = i / (2 * kWK);         // W slot sequence number
      const int r = (i >> 1) % kWK;        // unit within the slot
      const Slot ws(j, SW), as(i, SA);
      const int kt = kt_lo + (i >> 1), h = i & 1;
      mbar_wait_sleep(w_full(ws.s), ws.ph);
      if ((threadIdx.x & 127) == 0) TC_STAGE(i, 0);
      const uint32_t st = w_at(ws.s);
      LaneBits<BITS> lb[4];
      uint4 sq[4];
      if (active) {
        const uint32_t wr = st + u * kSlotW + r * kSubBytes;
        const int kt0 = kt_lo + j * kWK;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int kstep = q + 4 * h;  // k-step within the unit
          const int slot_u = kstep * 32 + lane;
          if constexpr (BITS == 4) {
            lb[q].w = lds128(wr + slot_u * 16);
          } else if constexpr (BITS == 2) {
            lb[q].w = lds64(wr + slot_u * 8);
          } else {
            lb[q].hi = lds64(wr + slot_u * 8);
            lb[q].lo = lds32(wr + 2048 + slot_u * 4);  // lane word C after words A, B
          }
          const int gl = (((kt << 7) + 16 * kstep) >> p.group_shift) - ((kt0 << 7) >> p.group_shift);
          sq[q] = lds128(st + 2 * kSlotW + u * p.ngw * 128 + gl * 128 + s_lane);
        }
      }
      if ((threadIdx.x & 127) == 0 && (reinterpret_cast<const uint32_t*>(&lb[0])[0] | sq[0].x) != 0x7fffffffu) TC_STAGE(i, 6);
      // this lane is done with the W slot after its group's last stage in it
      {
        const int slot_end = (j + 1) * 2 * kWK < nk ? (j + 1) * 2 * kWK : nk;
        if (i + kGroups >= slot_end) mbar_arrive(w_empty(ws.s));
      }
      if (i >= SA) mbar_wait_sleep(a_empty(as.s), as.ph ^ 1u);
      tmem_fence_after();
      if ((threadIdx.x & 127) == 0) TC_STAGE(i, 1);
      if (active) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int kl = q;  // k-step within the 64-k stage
#pragma unroll
          for (int jj = 0; jj < 2; ++jj) {
            const int jt = jb + jj;
            const uint32_t scw = jt == 0 ? sq[q].x : jt == 1 ? sq[q].y : jt == 2 ? sq[q].z : sq[q].w;
            uint32_t a[4];
            lut_dequant4_r128(atom_index_bytes<BITS>(lb[q], jt), lane8, lut, scw, a);
#ifdef FLUTE_DIAGNOSTICS
            if (p.diag & 1) continue;
#endif
            tmem_st_atom(t_lane + (static_cast<uint32_t>(16 * jj) << 16) + 32 * as.s + 8 * kl, a);
          }
        }
      }
      if ((threadIdx.x & 127) == 0) TC_STAGE(i, 4);
      tmem_wait_st();
      if ((threadIdx.x & 127) == 0) TC_STAGE(i, 5);
      tmem_fence_before();
      mbar_arrive(a_full(as.s));
      if ((threadIdx.x & 127) == 0) TC_STAGE(i, 2);
    }
    // ===================== epilogue (all 16 dequant warps) =====================
    // The accumulator (TMEM lane = output column n, column = row m) goes
    // through shared memory (the A / X rings are idle once every MMA has
    // completed) in chunks of 32 rows: warp w reads TMEM subpartition w % 4
    // (32 columns n) at rows [8 (w / 4), +8) of the chunk, then all 512
    // threads write the chunk's rows to global memory with 16-byte stores.
    mbar_wait_sleep(acc_full, 0);
    if (threadIdx.x == 0) TC_TRACE(1, tc_now());
    tmem_fence_after();
    {
      constexpr int kRows = 32;  // rows of m per chunk
      const bool f32 = p.splits > 1;
      const int esz = f32 ? 4 : 2;
      const uint32_t stage_buf = base + p.x_off;  // [kRows][128] elements (the idle X ring)
      const int sub = warp & 3;
      const int q8 = (warp >> 2) * 8;  // this warp's 8 rows of the chunk
      const int nl = sub * 32 + lane;  // column within the 128-column tile
      const int n0 = pair * 128;
      const int ncols = p.n - n0 < 128 ? p.n - n0 : 128;
      // accumulators written: one per issuer that had a stage
      const int nacc = nk < kNumAcc<BN> ? nk : kNumAcc<BN>;
      for (int c0 = 0; c0 < BN && m0 + c0 < p.m; c0 += kRows) {
        uint32_t v[8];
        for (int ja = 0; ja < nacc; ++ja) {
          uint32_t w[8];
          asm volatile(
              "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
              : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7])
              : "r"(tmem + (static_cast<uint32_t>(sub * 32) << 16) + static_cast<uint32_t>(ja * BN + c0 + q8))
              : "memory");
          tmem_wait_ld();
#pragma unroll
          for (int q = 0; q < 8; ++q)  // fixed accumulator order: bitwise reproducible
            v[q] = ja == 0 ? w[q] : __float_as_uint(__uint_as_float(v[q]) + __uint_as_float(w[q]));
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const uint32_t row = q8 + q;
          if (f32) {
            asm volatile("st.shared.u32 [%0], %1;" ::"r"(stage_buf + (row * 128 + nl) * 4), "r"(v[q]) : "memory");
          } else {
            const __half hv = __float2half_rn(__uint_as_float(v[q]));
            asm volatile("st.shared.u16 [%0], %1;" ::"r"(stage_buf + (row * 128 + nl) * 2),
                         "h"(*reinterpret_cast<const unsigned short*>(&hv))
                         : "memory");
          }
        }
        named_bar_sync(2, kDqWarps * 32);
        // rows of 128 * esz bytes, 16-byte chunks
        const int chunks_per_row = 128 * esz / 16;
        const int rows = p.m - (m0 + c0) < kRows ? p.m - (m0 + c0) : kRows;
        for (int idx = threadIdx.x; idx < rows * chunks_per_row; idx += kDqWarps * 32) {
          const int row = idx / chunks_per_row;
          const int ch = idx % chunks_per_row;
          const int col = ch * 16 / esz;  // first column of the chunk
          if (col >= ncols) continue;
          uint4 val;
          asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                       : "=r"(val.x), "=r"(val.y), "=r"(val.z), "=r"(val.w)
                       : "r"(stage_buf + row * 128 * esz + ch * 16));
          const size_t m = static_cast<size_t>(m0 + c0 + row);
          if (f32) {
            float* dst = p.part + (static_cast<size_t>(z) * p.m + m) * p.n + n0 + col;
            if (col + 4 <= ncols && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
              *reinterpret_cast<uint4*>(dst) = val;
            } else {
              const uint32_t e[4] = {val.x, val.y, val.z, val.w};
              for (int q = 0; q < 4 && col + q < ncols; ++q) dst[q] = __uint_as_float(e[q]);
            }
          } else {
            __half* dst = p.y + m * p.n + n0 + col;
            if (col + 8 <= ncols && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
              *reinterpret_cast<uint4*>(dst) = val;
            } else {
              const uint32_t e[4] = {val.x, val.y, val.z, val.w};
              const __half* h = reinterpret_cast<const __half*>(e);
              for (int q = 0; q < 8 && col + q < ncols; ++q) dst[q] = h[q];
            }
          }
        }
        named_bar_sync(2, kDqWarps * 32);
      }
    }
  }
  if (threadIdx.x == 0) TC_TRACE(2, tc_now());
  tmem_fence_before();
  __syncthreads();
  if (warp == kMmaWarp) {
    tmem_fence_after();
    tmem_dealloc(tmem, kTmemCols);
  }
}

// y[m][n] = f16(sum_z part[z][m][n]), z ascending (deterministic).
// Sums the split partials in fixed split order and re-zeroes them: the
// workspace is shared with the Stream-K path, whose slots must read zero
// ("unwritten") at rest (qgemm_kernel.cuh fixup protocol).
// (only when the partials live in that shared workspace: ZERO).
template <bool ZERO>
__global__ void splitk_reduce_kernel(float* __restrict__ part, __half* __restrict__ y, int splits,
                                     size_t mn) {
  pdl_wait();
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < mn;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    float acc = part[i];
    for (int z = 1; z < splits; ++z) acc += part[static_cast<size_t>(z) * mn + i];
    y[i] = __float2half_rn(acc);
    if (ZERO)
      for (int z = 0; z < splits; ++z) part[static_cast<size_t>(z) * mn + i] = 0.f;
  }
}

}  // namespace tc

namespace {

[[noreturn]] void tc_fail(const char* what, cudaError_t e) {
  throw flutesim::CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}
#define FLUTE_TC_CUDA(call)                         \
  do {                                              \
    cudaError_t e_ = (call);                        \
    if (e_ != cudaSuccess) tc_fail(#call, e_);      \
  } while (0)

using EncodeTiledTc = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledTc encode_tc() {
  static EncodeTiledTc fn = [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || ptr == nullptr)
      throw flutesim::CudaError("cuTensorMapEncodeTiled entry point unavailable");
    return reinterpret_cast<EncodeTiledTc>(ptr);
  }();
  return fn;
}

struct TcPlan {
  int bn = 128, splits = 1, stages = 2;
  bool zero_part = false;
  size_t smem = 0;
  tc::Params prm{};
};

template <int BITS, int BN>
void launch_tc(const GemmArgs& a, const TcPlan& pl, cudaStream_t stream) {
  static thread_local int configured = -1;
  int dev = 0;
  FLUTE_TC_CUDA(cudaGetDevice(&dev));
  auto kern = tc::qgemm_tc_kernel<BITS, BN>;
  if (configured != dev) {
    int optin = 0;
    FLUTE_TC_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    FLUTE_TC_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, optin));
    configured = dev;
  }
  CUtensorMap map;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(a.k), static_cast<cuuint64_t>(a.m)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(a.k) * 2};
  const cuuint32_t box[2] = {64u, static_cast<cuuint32_t>(BN)};
  const cuuint32_t estr[2] = {1u, 1u};
  const CUresult r = encode_tc()(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void*>(a.x),
                                 dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                 CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    throw flutesim::InputError("X tensor map rejected (x must be 16-byte aligned, k % 8 == 0)");
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(pl.prm.tiles_n + 1) / 2,
                     static_cast<unsigned>((a.m + BN - 1) / BN), static_cast<unsigned>(pl.splits));
  cfg.blockDim = dim3(tc::threads_for_bn(pl.bn));
  cfg.dynamicSmemBytes = pl.smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
#ifdef FLUTE_DIAGNOSTICS
  // FLUTE_TC_TRACE=file: per-CTA / per-stage timeline of this launch (sync)
  const char* trace_path = std::getenv("FLUTE_TC_TRACE");
  tc::Params prm = pl.prm;
  prm.diag = std::getenv("FLUTE_TC_DIAG") ? std::atoi(std::getenv("FLUTE_TC_DIAG")) : 0;
  unsigned long long* tr = nullptr;
  const size_t ctas = static_cast<size_t>(cfg.gridDim.x) * cfg.gridDim.y * cfg.gridDim.z;
  const size_t words = ctas * 4 + ctas * 64 * 8;
  if (trace_path) {
    FLUTE_TC_CUDA(cudaMalloc(&tr, words * 8));
    FLUTE_TC_CUDA(cudaMemset(tr, 0, words * 8));
    prm.trace = tr;
  }
  FLUTE_TC_CUDA(cudaLaunchKernelEx(&cfg, kern, map, prm));
  if (trace_path) {
    FLUTE_TC_CUDA(cudaDeviceSynchronize());
    std::vector<unsigned long long> h(words);
    FLUTE_TC_CUDA(cudaMemcpy(h.data(), tr, words * 8, cudaMemcpyDeviceToHost));
    cudaFree(tr);
    if (FILE* f = std::fopen(trace_path, "wb")) {
      const unsigned long long hdr[2] = {ctas, 64};
      std::fwrite(hdr, 8, 2, f);
      std::fwrite(h.data(), 8, words, f);
      std::fclose(f);
    }
  }
#else
  FLUTE_TC_CUDA(cudaLaunchKernelEx(&cfg, kern, map, pl.prm));
#endif
  if (pl.splits > 1) {
    const size_t mn = static_cast<size_t>(a.m) * a.n;
    cudaLaunchConfig_t c2{};
    c2.gridDim = dim3(static_cast<unsigned>(std::min<size_t>((mn + 255) / 256, 148 * 8)));
    c2.blockDim = dim3(256);
    c2.stream = stream;
    c2.attrs = attr;
    c2.numAttrs = 1;
    if (pl.zero_part)
      FLUTE_TC_CUDA(cudaLaunchKernelEx(&c2, tc::splitk_reduce_kernel<true>, pl.prm.part,
                                       static_cast<__half*>(a.y), pl.splits, mn));
    else
      FLUTE_TC_CUDA(cudaLaunchKernelEx(&c2, tc::splitk_reduce_kernel<false>, pl.prm.part,
                                       static_cast<__half*>(a.y), pl.splits, mn));
  }
}

}  // namespace

// X rows per CTA: 64 / 128, or 256 (UMMA N = 256 with 64-deep stages) when
// 128-row tiles would need more than one wave of CTAs — each dequantised W^T
// tile then feeds twice as many rows (measured: 8192^2 M=512 123 -> 79 us;
// with a single wave of 128-row tiles BN = 128 stays faster, e.g. 4096^2
// M=512 34 vs 38 us, because BN = 256 would then need split-K).
int tc_bn(int m, int tiles_n, int sms) {
  if (std::getenv("FLUTE_TC_BN")) return std::atoi(std::getenv("FLUTE_TC_BN"));
  if (m <= 32) return 32;
  if (m < 128) return 64;
  const long tiles128 = static_cast<long>((tiles_n + 1) / 2) * ((m + 127) / 128);
  return m >= 256 && tiles128 > sms ? 256 : 128;
}

size_t tc_workspace_bytes(int m, int k, int n, int sms) {
  const int tiles_n = (n + 63) / 64;
  const int tiles_k = (k + 127) / 128;
  const int bn = tc_bn(m, tiles_n, sms);
  const long tiles = static_cast<long>((tiles_n + 1) / 2) * ((m + bn - 1) / bn);
  int splits = static_cast<int>(std::max<long>(1, std::min<long>(std::min(tiles_k, 8), sms / std::max<long>(tiles, 1))));
  if (const char* f = std::getenv("FLUTE_TC_SPLITS")) splits = std::max(1, std::min(tiles_k, std::atoi(f)));
  return splits > 1 ? static_cast<size_t>(splits) * m * n * 4 : 0;
}

// Rows from which the tcgen05 kernel takes over from the mma.sync kernel
// (FLUTE_TC_MIN_M overrides, for measurements).
bool tc_enabled(int m) {
  const char* e = std::getenv("FLUTE_TC_MIN_M");  // (read per call: tests switch it)
  const int min_m = e ? std::atoi(e) : 64;
  return m >= min_m && std::getenv("FLUTE_NO_TC") == nullptr;
}

void qgemm_tc(const GemmArgs& a, int tiles_k, int tiles_n, int gp, int sms, bool zero_part,
              void* part, size_t part_bytes) {
  TcPlan pl;
  pl.zero_part = zero_part;
  pl.bn = tc_bn(a.m, tiles_n, sms);
  if (pl.bn != 32 && pl.bn != 64 && pl.bn != 128 && pl.bn != 256)
    throw flutesim::ConfigError("FLUTE_TC_BN must be 32, 64, 128 or 256");
  const long tiles = static_cast<long>((tiles_n + 1) / 2) * ((a.m + pl.bn - 1) / pl.bn);
  pl.splits = static_cast<int>(
      std::max<long>(1, std::min<long>(std::min(tiles_k, 8), sms / std::max<long>(tiles, 1))));
  if (const char* f = std::getenv("FLUTE_TC_SPLITS")) pl.splits = std::max(1, std::min(tiles_k, std::atoi(f)));
  while (pl.splits > 1 && static_cast<size_t>(pl.splits) * a.m * a.n * 4 > part_bytes) --pl.splits;
  // [vLUT | barriers | X ring (sx x BN*128) | W ring (sw x w_stage)]; the A
  // ring (sa slots of 32 columns) is in tensor memory
  const int ngw = tc::kWK * 128 / a.group + 1;  // + 1: a slot may start mid-group (g = 256)
  const size_t lut = static_cast<size_t>(kTableRows<4>) * 128;  // compact vLUT (128-byte rows, 256 of them)
  const size_t bar_off = lut;
  const size_t x_off = (bar_off + 8 * (2 * tc::kMaxW + 2 * tc::kMaxA + 2 * tc::kMaxX + 2) + 1023) / 1024 * 1024;
  const size_t x_bytes = static_cast<size_t>(pl.bn) * 128;
  const size_t w_stage = (2 * static_cast<size_t>(tc::kWK) * a.bits * 1024 + 2 * static_cast<size_t>(ngw) * 128 +
                           127) / 128 * 128;
  int optin = 0, dev = 0;
  FLUTE_TC_CUDA(cudaGetDevice(&dev));
  FLUTE_TC_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  // ring depths (shared memory): at least X 2 / W 3, then X up to 4 slots
  // (8 while they stay within 64 KB), then W up to 8 slots
  auto used = [&](int sx_, int sw_) { return x_off + sx_ * x_bytes + sw_ * w_stage; };
  const size_t cap = static_cast<size_t>(optin);
  int sx = 2, sw = 3;
  if (used(sx, sw) > cap) throw flutesim::InternalError("qgemm_tc: shared-memory plan does not fit");
  while (sx < tc::kMaxX && (sx < 4 || (sx + 1) * x_bytes <= 64 * 1024) && used(sx + 1, sw) <= cap) ++sx;
  while (sw < tc::kMaxW && used(sx, sw + 1) <= cap) ++sw;
  // the A ring (tensor memory, <= kMaxA x 32 columns above the accumulator)
  // pairs slot for slot with the X ring: one release barrier per pair
  // A ring in tensor memory: kMaxA x 32 columns above the accumulators.
  // Stage i is dequantised by group i % 4 into A slot i % sa (sa = 8: each group
  // alternates between two slots, dequantising a stage while the MMAs of
  // its previous one still read the other); a slot's phases are always waited
  // by the same group, in order.  The MMAs of a stage release its A slot and
  // (BN < 256) its X slot; at BN = 256 X slot s is reused after the A release
  // of the stage SX earlier.
  // (BN = 256: four slots, one per group — its 128-cycle UMMAs keep the
  // tensor pipe busy and a deeper A ring only adds TMEM traffic, measured
  // 54 -> 61 us at 8192^2 M=512)
  static_assert(tc::kMaxA % tc::kGroups == 0, "A slots shared evenly by the dequant groups");
  const int sa = pl.bn >= 256 ? tc::kGroups : tc::kMaxA;
  if (pl.bn >= 256 && sx > sa) sx = sa;  // (BN = 256: X slots tracked through the A-ring releases)
  // the epilogue stages 32 fp32 rows x 128 columns through the idle X ring
  if (static_cast<size_t>(sx) * x_bytes < 32 * 128 * 4)
    throw flutesim::InternalError("qgemm_tc: X ring smaller than the epilogue staging buffer");
  const size_t w_off = x_off + sx * x_bytes;
  pl.stages = sw;
  pl.smem = w_off + sw * w_stage;
  if (std::getenv("FLUTE_TC_PLAN"))  // measurement aid: print the ring plan
    std::fprintf(stderr, "qgemm_tc m=%d k=%d n=%d bits=%d: BN=%d splits=%d sw=%d sx=%d sa=%d smem=%zu w_stage=%zu\n",
                 a.m, a.k, a.n, a.bits, pl.bn, pl.splits, sw, sx, sa, pl.smem, w_stage);
  tc::Params& p = pl.prm;
  p.w = static_cast<const uint8_t*>(a.w);
  p.sc = static_cast<const uint8_t*>(a.scales);
  p.vlut = static_cast<const uint32_t*>(a.vlut);
  p.y = static_cast<__half*>(a.y);
  p.part = static_cast<float*>(part);
  p.m = a.m;
  p.n = a.n;
  p.tiles_k = tiles_k;
  p.tiles_n = tiles_n;
  p.gp = gp;
  p.group_shift = __builtin_ctz(static_cast<unsigned>(a.group));
  p.splits = pl.splits;
  p.sw = sw;
  p.sx = sx;
  p.sa = sa;
  p.ngw = ngw;
  p.bar_off = static_cast<uint32_t>(bar_off);
  p.x_off = static_cast<uint32_t>(x_off);
  p.w_off = static_cast<uint32_t>(w_off);
  p.w_stage = static_cast<uint32_t>(w_stage);
  cudaStream_t st = static_cast<cudaStream_t>(a.stream);
  auto go = [&](auto bits_tag) {
    constexpr int B = decltype(bits_tag)::value;
    if (pl.bn == 256) launch_tc<B, 256>(a, pl, st);
    else if (pl.bn == 128) launch_tc<B, 128>(a, pl, st);
    else if (pl.bn == 64) launch_tc<B, 64>(a, pl, st);
    else launch_tc<B, 32>(a, pl, st);
  };
  switch (a.bits) {
    case 2: go(std::integral_constant<int, 2>{}); break;
    case 3: go(std::integral_constant<int, 3>{}); break;
    default: go(std::integral_constant<int, 4>{}); break;
  }
}

}  // namespace flute_dev
