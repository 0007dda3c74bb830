// flute-b200 — the LUT-dequant Stream-K GEMM for the memory-bound regime
// (M <= 64 rows of X per launch), sm_100a, on the 5th-generation tensor cores
// with the dequantised weights as a TENSOR-MEMORY operand ("TS" MMA).
// Host launcher: qgemm_ts.cu.
//
// Reference semantics: flutesim::execute (engine.cpp:345) — Y = X * W_hat with
// W_hat = f16(scale * T[index]) (vec_lut.cpp:39-48) and fp32 accumulation;
// Stream-K ranges [floor(w*U/P), floor((w+1)*U/P)) over 64x128 units (n-tile
// major, k inner; streamk.cpp:17-58) with a fixed-order fixup of split tiles
// (engine.cpp:279-333).
//
// Why tensor memory: the weights are dequantised in registers (vLUT lookups in
// shared memory) and the registers go straight to TMEM with tcgen05.st — the
// A-fragment register pattern of the device layout IS the 16x128b store
// pattern — so neither an STS of W^T nor an HMMA per 16x16 atom is needed: one
// thread issues tcgen05.mma (A = W^T from TMEM, M = 64; B = X^T from shared
// memory, N = NB = 8/16/32/64; D fp32 in TMEM) for a whole 64x16 k-step.  The
// dequant warps touch shared memory only for the packed words and the vLUT
// lookups, and TMEM holds up to 15 units of dequantised weights, so dequant
// runs ahead of X (which arrives only after the programmatic-dependent-launch
// wait) and the accumulators never occupy registers.
//
// Tensor-memory map (512 columns x 128 lanes, one CTA per SM).  M = 64 uses
// the low 16 lanes of every 32-lane subpartition; the high 16 lanes form a
// second, independent 64-row space ("half" h = 1).  Quad h (k-steps 4h..4h+3)
// of every unit goes to half h, so each unit feeds both halves and the two
// halves' accumulators are added in the epilogue:
//   D buffer b (b = tile sequence parity): columns [b*NB, b*NB + NB), both halves
//   A slot a (one unit, 8 k-steps):        columns [A0 + 32a, A0 + 32a + 32):
//       half h, column A0 + 32a + 8c = k-step 4h + c (16 k = 8 f16 pairs)
//   row r of a 64-row tile (output column 16q + i) -> lane 32q + 16h + i.
//
// Warp roles (threads = 32 * (6 + DW)):
//   0..3  epilogue (warp q reads TMEM subpartition q): D -> registers, halves
//         added, Stream-K / cluster split-K reduction, Y (+ peer copies)
//   4     producer: per stage one bulk copy of the weights (UBLKCP, evict-first),
//         one of the scales, one 3-D TMA box of X (128B swizzle); the first S
//         stages' weights/scales are issued BEFORE griddepcontrol.wait
//   5     MMA issuer (+ TMEM alloc/dealloc)
//   6..   DW dequant warps: warp w owns TMEM subpartition q = w & 3 (the atom
//         = 16 output columns it may write) and takes the (unit, quad) items of
//         that atom round-robin with the other DW/4 warps of its subpartition.
#pragma once

#include <cuda.h>
#include <cuda_fp16.h>

#include "dequant.cuh"
#include "ptx.cuh"

namespace flute_dev {
namespace ts {

constexpr int kUnitN = 64;   // == flutesim::kUnitN
constexpr int kUnitK = 128;  // == flutesim::kUnitK
constexpr int kMaxStages = 16;
constexpr int kMaxPeers = 8;
constexpr int kEpiWarps = 4, kProducerWarp = 4, kMmaWarp = 5, kFirstDqWarp = 6;
constexpr int threads_for(int dw) { return 32 * (kFirstDqWarp + dw); }

// TMEM plan for an NB-row launch
template <int NB>
struct TmemPlan {
  static constexpr int kA0 = (2 * NB + 31) / 32 * 32;  // first A column
  static constexpr int kSlots = (512 - kA0) / 32 < 16 ? (512 - kA0) / 32 : 16;
};

struct Params {
  const uint8_t* w;
  const uint8_t* sc;
  const uint32_t* vlut;
  // Output: every value is stored to y_out[0..n_out) at [row * ldy + ycol0 + col]
  // (n_out > 1: the N-sharded layer's all-gather fused into the epilogue).
  __half* y_out[kMaxPeers];
  int n_out, ldy, ycol0;
  float* slots;      // Stream-K partials, [worker][NB][64] fp32 (bit-inverted)
  uint32_t* flags;   // [workers] unused, [workers] ticket, [workers+1] done count
  int m, n;
  int tiles_k;       // units per 64-column tile
  int group_shift;   // log2(group size)
  int gp;            // padded groups per column
  int units;
  int workers;
  int stages;
  int ups;           // units per stage
  int use_ticket;
  int x3d;           // X tensor map is the 3-D {64, m, k/64} view (k % 64 == 0)
  int cluster;       // > 1: cluster split-K (cluster c = tile c, k split C ways)
  uint32_t bar_off, recv_off, stage_off, stage_bytes, x_bytes, w_bytes;
};

// ---- tcgen05 helpers ---------------------------------------------------------
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// K-major, 128B swizzle, 8-row groups 1024 B apart (sm_100 descriptor v1).
__device__ __forceinline__ uint64_t desc_sw128(uint32_t addr) {
  return static_cast<uint64_t>((addr >> 4) & 0x3FFFu) | (static_cast<uint64_t>(1) << 16) |
         (static_cast<uint64_t>(1024 >> 4) << 32) | (static_cast<uint64_t>(1) << 46) |
         (static_cast<uint64_t>(2) << 61);
}
// kind::f16, D f32, A/B f16 K-major, M = 64, N = nb.
__host__ __device__ constexpr uint32_t idesc_m64(int nb) {
  return (1u << 4) | (static_cast<uint32_t>(nb >> 3) << 17) | (static_cast<uint32_t>(64 >> 4) << 24);
}
__device__ __forceinline__ void umma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                        uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void umma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
               : "memory");
}
// 16 lanes x 32 columns from the A-fragment registers of 4 k-steps
// (rep r = columns 4r..4r+3 from registers 2r, 2r+1).
__device__ __forceinline__ void tmem_st_16x128_x8(uint32_t taddr, const uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.16x128b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, "
      "%12, %13, %14, %15, %16};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
      "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
// thread = TMEM lane (32 lanes of the warp's subpartition), 8 consecutive columns
// (the registers are valid only after tmem_ld_wait)
__device__ __forceinline__ void tmem_ld_32x32_x8(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
      : "r"(taddr)
      : "memory");
}
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// Host guarantees units * (workers + 1) < 2^31, so 32-bit math is exact.
__device__ __forceinline__ int range_lo(int w, int U, int P) {
  return static_cast<int>(static_cast<uint32_t>(U) * static_cast<uint32_t>(w) / static_cast<uint32_t>(P));
}
__device__ __forceinline__ int owner_of(int x, int U, int P) {
  int w = static_cast<int>(static_cast<uint32_t>(x) * static_cast<uint32_t>(P) / static_cast<uint32_t>(U));
  if (w >= P) w = P - 1;
  while (w + 1 < P && range_lo(w + 1, U, P) <= x) ++w;
  while (w > 0 && range_lo(w, U, P) > x) --w;
  return w;
}

// The CTA's range [ubeg, uend) as segments (one per tile, walked in
// descending tile order: a split tile's contributor segment is processed —
// and published — first, so its finisher rarely waits).
struct SegRange {
  int t_hi, t_lo, ubeg, uend, tiles_k;
  __device__ __forceinline__ void init(int ub, int ue, int tk) {
    ubeg = ub;
    uend = ue;
    tiles_k = tk;
    t_hi = (ue - 1) / tk;
    t_lo = ub / tk;
  }
  __device__ __forceinline__ int top(int t) const { return t == t_hi ? uend - 1 - t * tiles_k : tiles_k - 1; }
  __device__ __forceinline__ int bot(int t) const { return t == t_lo ? ubeg - t * tiles_k : 0; }
};

// Walks the CTA's stages in the one order every role uses: tiles descending,
// inside a tile stages of up to `ups` units from the top k-slice down, units
// of a stage ascending.  fn(tile, lo, ns, first_of_tile, last_of_tile).
template <class F>
__device__ __forceinline__ void walk_stages(const SegRange& R, int ups, F&& fn) {
  if (R.uend <= R.ubeg) return;
  for (int t = R.t_hi; t >= R.t_lo; --t) {
    const int bot = R.bot(t);
    const int top = R.top(t);
    for (int kt = top; kt >= bot; kt -= ups) {
      const int lo = kt - ups + 1 > bot ? kt - ups + 1 : bot;
      fn(t, lo, kt - lo + 1, kt == top, lo == bot);
    }
  }
}

template <int BITS, int NB, int DW>
__global__ void __launch_bounds__(threads_for(DW), 1)
    qgemm_ts_kernel(const __grid_constant__ CUtensorMap tmap_x, const Params p) {
  using TP = TmemPlan<NB>;
  constexpr int kSubBytes = BITS * 1024;  // one unit's packed weights
  constexpr int R = DW / 4;               // dequant warps per TMEM subpartition
  extern __shared__ __align__(1024) uint8_t smem[];

  const int S = p.stages;
  const uint32_t base = smem_u32(smem);
  const uint32_t lut = base;
  const uint32_t bars = base + p.bar_off;
  auto w_full = [&](int s) { return bars + 8 * s; };
  auto x_full = [&](int s) { return bars + 8 * (kMaxStages + s); };
  auto empty = [&](int s) { return bars + 8 * (2 * kMaxStages + s); };
  auto a_full = [&](int a) { return bars + 8 * (3 * kMaxStages + a); };
  auto a_empty = [&](int a) { return bars + 8 * (4 * kMaxStages + a); };
  auto d_full = [&](int b) { return bars + 8 * (5 * kMaxStages + b); };
  auto d_empty = [&](int b) { return bars + 8 * (5 * kMaxStages + 2 + b); };
  const uint32_t recv_bar = bars + 8 * (5 * kMaxStages + 4);
  uint32_t* misc = reinterpret_cast<uint32_t*>(smem + p.bar_off + 8 * (5 * kMaxStages + 5));
  // misc[0]: TMEM base, misc[1]: ticket
  auto xs_of = [&](int s) { return base + p.stage_off + s * p.stage_bytes; };
  auto ws_of = [&](int s) { return xs_of(s) + p.x_bytes; };
  auto ss_of = [&](int s) { return xs_of(s) + p.x_bytes + p.w_bytes; };

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(w_full(s), 1);
      mbar_init(x_full(s), 1);
      mbar_init(empty(s), DW + 1);  // every dequant warp + the MMA commit
    }
    for (int a = 0; a < TP::kSlots; ++a) {
      mbar_init(a_full(a), 8);  // 4 subpartitions x 2 quads
      mbar_init(a_empty(a), 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(d_full(b), 1);
      mbar_init(d_empty(b), kEpiWarps);
    }
    if (p.cluster > 1) mbar_init(recv_bar, 32 * kEpiWarps * (p.cluster - 1));
    fence_mbar_init();
  }
  if (warp == kMmaWarp) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     smem_u32(&misc[0]))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  int wid = blockIdx.x;
  if (p.use_ticket) {
    // More workers than co-resident CTAs: take worker ids in start order so a
    // finisher only ever waits on CTAs that are already running.
    pdl_wait();
    if (threadIdx.x == 0) misc[1] = atomicAdd(p.flags + p.workers, 1u);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = misc[0];
  if (p.use_ticket) wid = static_cast<int>(misc[1]);
  if (p.cluster > 1) cluster_arrive_relaxed();  // recv barrier initialised before any peer arrives
  pdl_launch_dependents();

  const int U = p.units;
  const int P = p.workers;
  const int tiles_k = p.tiles_k;
  int ubeg, uend;
  uint32_t crank = 0;
  if (p.cluster > 1) {
    crank = cluster_ctarank();
    const int t0c = static_cast<int>(cluster_id_x()) * tiles_k;
    ubeg = t0c + static_cast<int>(crank) * tiles_k / p.cluster;
    uend = t0c + (static_cast<int>(crank) + 1) * tiles_k / p.cluster;
  } else {
    ubeg = range_lo(wid, U, P);
    uend = range_lo(wid + 1, U, P);
  }
  const int gshift = p.group_shift;
  SegRange Rg;
  Rg.init(ubeg, uend, tiles_k);

  if (warp == kProducerWarp) {
    // ===================== producer =====================
    if (uend > ubeg) {
      const bool leader = elect_one();
      if (leader) prefetch_tmap(&tmap_x);
      const uint64_t pol = policy_evict_first();
      auto issue_ws = [&](int t, int lo, int ns, int s) {
        const int glo = (lo * kUnitK) >> gshift;
        const int ng = ((((lo + ns) * kUnitK) - 1) >> gshift) - glo + 1;
        if (leader) {
          mbar_arrive_expect_tx(w_full(s), ns * kSubBytes + ng * 128);
          bulk_g2s_hint(ws_of(s), p.w + static_cast<size_t>(t * tiles_k + lo) * kSubBytes, ns * kSubBytes,
                        w_full(s), pol);
          bulk_g2s(ss_of(s), p.sc + (static_cast<size_t>(t) * p.gp + glo) * 128, ng * 128, w_full(s));
        }
      };
      auto issue_x = [&](int lo, int ns, int s) {
        if (!leader) return;
        if (p.x3d) {
          mbar_arrive_expect_tx(x_full(s), 2 * p.ups * NB * 128);
          tma_3d_g2s(xs_of(s), &tmap_x, 0, 0, lo * 2, x_full(s));
        } else {
          mbar_arrive_expect_tx(x_full(s), 2 * ns * NB * 128);
          for (int c = 0; c < 2 * ns; ++c)
            tma_2d_g2s(xs_of(s) + c * NB * 128, &tmap_x, lo * kUnitK + 64 * c, 0, x_full(s));
        }
      };
      // pass 1 (before the PDL wait): weights + scales of the first S stages
      int pre = 0;
      walk_stages(Rg, p.ups, [&](int t, int lo, int ns, bool, bool) {
        if (pre < S) issue_ws(t, lo, ns, pre);
        ++pre;
      });
      if (pre > S) pre = S;
      if (!p.use_ticket) pdl_wait();  // X belongs to the previous kernel in the stream
      int it = 0;
      walk_stages(Rg, p.ups, [&](int t, int lo, int ns, bool, bool) {
        const int s = it % S;
        const uint32_t ph = static_cast<uint32_t>(it / S) & 1u;
        if (it >= pre) {
          mbar_wait_sleep(empty(s), ph ^ 1u);
          issue_ws(t, lo, ns, s);
        }
        issue_x(lo, ns, s);
        ++it;
      });
    }
  } else if (warp == kMmaWarp) {
    // ===================== MMA issuer =====================
    constexpr uint32_t idesc = idesc_m64(NB);
    int it = 0, j = 0, tseq = 0;
    walk_stages(Rg, p.ups, [&](int, int, int ns, bool first_of_tile, bool last_of_tile) {
      const int s = it % S;
      const uint32_t ph = static_cast<uint32_t>(it / S) & 1u;
      const int b = tseq & 1;
      if (first_of_tile && tseq >= 2) mbar_wait(d_empty(b), ((tseq >> 1) & 1) ^ 1);
      mbar_wait(x_full(s), ph);
      for (int i = 0; i < ns; ++i, ++j) {
        const int a = j % TP::kSlots;
        mbar_wait(a_full(a), static_cast<uint32_t>(j / TP::kSlots) & 1u);
        tc_fence_after();
        if (elect_one()) {
          const bool fresh = first_of_tile && i == 0;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const uint32_t hl = static_cast<uint32_t>(16 * h) << 16;
            const uint32_t xb = xs_of(s) + (2 * i + h) * NB * 128;
#pragma unroll
            for (int c = 0; c < 4; ++c)
              umma_ts(tmem + hl + b * NB, tmem + hl + TP::kA0 + 32 * a + 8 * c, desc_sw128(xb + 32 * c), idesc,
                      (fresh && c == 0) ? 0u : 1u);
          }
          umma_commit(a_empty(a));  // A slot free once these MMAs have read it
          if (last_of_tile && i == ns - 1) umma_commit(d_full(b));
        }
        __syncwarp();
      }
      if (elect_one()) umma_commit(empty(s));  // X of the stage read
      __syncwarp();
      if (last_of_tile) ++tseq;
      ++it;
    });
  } else if (warp >= kFirstDqWarp) {
    // ===================== dequant warps =====================
    fill_lut<BITS, DW * 32>(lut, p.vlut, threadIdx.x - kFirstDqWarp * 32);
    named_bar_sync(1, DW * 32);
    const int q = warp & 3;                    // TMEM subpartition = atom (16 columns)
    const int r = (warp - kFirstDqWarp) >> 2;  // rank among this subpartition's warps
    const uint32_t lane4 = static_cast<uint32_t>(lane) * 4u;
    const uint32_t s_lane = (lane >> 2) * 16 + q * 4;
    int it = 0, j = 0;
    walk_stages(Rg, p.ups, [&](int, int lo, int ns, bool, bool) {
      const int s = it % S;
      const uint32_t ph = static_cast<uint32_t>(it / S) & 1u;
      const int glo = (lo * kUnitK) >> gshift;
      // every warp waits for the stage (even without items in it): its arrive
      // on empty(s) below must not run ahead into the slot's previous phase
      mbar_wait(w_full(s), ph);
      for (int item = 0; item < 2 * ns; ++item) {
        if (item % R != (r + j) % R) continue;  // rotate the start so the load spreads
        const int i = item >> 1, h = item & 1;
        const int ju = j + i;
        const uint32_t wu = ws_of(s) + i * kSubBytes;
        const int slot = (h * 4 + q) * 32 + lane;
        LaneBits<BITS> lb;
        if constexpr (BITS == 4) {
          lb.w = lds128(wu + slot * 16);
        } else if constexpr (BITS == 2) {
          lb.w = lds64(wu + slot * 8);
        } else {
          lb.hi = lds64(wu + slot * 8);
          lb.lo = lds32(wu + 2048 + slot * 4);
        }
        const int k0 = (lo + i) * kUnitK + 64 * h;
        const uint32_t sb = ss_of(s) + s_lane;
        const uint32_t sc0 = lds32(sb + ((k0 >> gshift) - glo) * 128);
        const uint32_t sc1 = lds32(sb + (((k0 + 32) >> gshift) - glo) * 128);
        uint32_t a[16];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint32_t v[4];
          lut_dequant4(word_index_bytes<BITS>(lb, c), lane4, lut, c < 2 ? sc0 : sc1, v);
#pragma unroll
          for (int pp = 0; pp < 4; ++pp) a[4 * c + pp] = v[pp];
        }
        const int as = ju % TP::kSlots;
        mbar_wait(a_empty(as), (static_cast<uint32_t>(ju / TP::kSlots) & 1u) ^ 1u);
        tc_fence_after();
        tmem_st_16x128_x8(tmem + (static_cast<uint32_t>(32 * q + 16 * h) << 16) + TP::kA0 + 32 * as, a);
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(a_full(as));
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(empty(s));  // this warp is done with the stage's weights
      j += ns;
      ++it;
    });
  } else {
    // ===================== epilogue warps 0..3 =====================
    const int q = warp;
    if (!p.use_ticket) pdl_wait();  // the workspace and Y belong to the previous kernel
    int tseq = 0;
    for (int tile = Rg.t_hi; uend > ubeg && tile >= Rg.t_lo; --tile, ++tseq) {
      const int b = tseq & 1;
      mbar_wait_sleep(d_full(b), (tseq >> 1) & 1);
      tc_fence_after();
      uint32_t raw[NB];
#pragma unroll
      for (int c0 = 0; c0 < NB; c0 += 8)
        tmem_ld_32x32_x8(tmem + (static_cast<uint32_t>(32 * q) << 16) + b * NB + c0, raw + c0);
      tmem_ld_wait();
      float acc[NB];
#pragma unroll
      for (int i = 0; i < NB; ++i) acc[i] = __uint_as_float(raw[i]);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(d_empty(b));
      // lanes 0..15: half 0 of column 16q + lane; lanes 16..31: half 1 of it
#pragma unroll
      for (int i = 0; i < NB; ++i) acc[i] += __shfl_down_sync(0xffffffffu, acc[i], 16);
      const bool act = lane < 16;
      const int colt = 16 * q + lane;  // column within the 64-column tile
      const int t0 = tile * tiles_k;
      const bool started = ubeg <= t0;
      const bool finished = uend >= t0 + tiles_k;
      const int mrows = p.m < NB ? p.m : NB;
      if (p.cluster > 1) {
        // ---- cluster split-K: ranks > 0 push their partial into rank 0's
        // receive buffer through DSMEM; rank 0 adds them in rank order ----
        const uint32_t recv = base + p.recv_off;
        cluster_wait();  // every CTA has initialised its barriers
        if (crank != 0) {
          if (act) {
            const uint32_t dst = mapa_shared(recv + ((crank - 1) * NB * 64 + colt) * 4, 0);
            for (int i = 0; i < mrows; ++i) st_cluster_f32(dst + i * 256, acc[i]);
          }
          mbar_arrive_remote(mapa_shared(recv_bar, 0));
          continue;
        }
        mbar_wait_cluster(recv_bar, 0);
        for (int rr = 1; rr < p.cluster; ++rr) {
#pragma unroll
          for (int i = 0; i < NB; ++i) {
            if (i < mrows && act) {
              float v;
              asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(recv + (((rr - 1) * NB + i) * 64 + colt) * 4));
              acc[i] += v;
            }
          }
        }
      } else if (!finished) {
        // contributor: publish the fp32 partial as bit-inverted words, so an
        // all-zero slot means "not written yet" (0xFFFFFFFF is never produced:
        // NaNs are canonicalised to 0x7FFFFFFF).  No flag, no fence: the
        // finisher polls the data itself.
        if (act) {
          volatile uint32_t* my = reinterpret_cast<volatile uint32_t*>(p.slots) +
                                  static_cast<size_t>(wid) * NB * 64 + colt;
#pragma unroll
          for (int i = 0; i < NB; ++i) {
            if (i < mrows) {
              uint32_t bits = __float_as_uint(acc[i]);
              if (bits == 0xFFFFFFFFu) bits = 0x7FFFFFFFu;
              my[i * 64] = ~bits;
            }
          }
        }
        continue;
      } else if (!started) {
        // finisher: contributors = non-empty workers in [owner(t0), wid), added
        // to the own partial in ascending worker (= ascending k) order — a
        // fixed order, so results are bitwise reproducible.
        const int first = owner_of(t0, U, P);
        for (int c = first; c < wid; ++c) {
          if (range_lo(c + 1, U, P) <= range_lo(c, U, P)) continue;
          if (!act) continue;
          volatile uint32_t* src = reinterpret_cast<volatile uint32_t*>(p.slots) +
                                   static_cast<size_t>(c) * NB * 64 + colt;
#pragma unroll
          for (int i0 = 0; i0 < NB; i0 += 8) {
            if (i0 >= mrows) break;
            uint32_t v[8];
            bool ready;
            do {
              ready = true;
#pragma unroll
              for (int i = 0; i < 8; ++i) {
                v[i] = i0 + i < mrows ? src[(i0 + i) * 64] : 1u;
                ready &= v[i] != 0u;
              }
            } while (!ready);
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              if (i0 + i < mrows) {
                acc[i0 + i] += __uint_as_float(~v[i]);
                src[(i0 + i) * 64] = 0u;  // re-arm (graph / back-to-back safe)
              }
            }
          }
        }
      }
      // write Y (f16, RNE)
      const int col = tile * kUnitN + colt;
      if (act && col < p.n) {
#pragma unroll 1
        for (int d = 0; d < p.n_out; ++d) {
          __half* yb = p.y_out[d] + p.ycol0 + col;
#pragma unroll
          for (int i = 0; i < NB; ++i)
            if (i < mrows) yb[static_cast<size_t>(i) * p.ldy] = __float2half_rn(acc[i]);
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarp) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
  if (p.use_ticket && threadIdx.x == 0) {
    __threadfence();
    const uint32_t done = atomicAdd(p.flags + p.workers + 1, 1u);
    if (done == static_cast<uint32_t>(P) - 1u) {
      p.flags[p.workers] = 0u;
      p.flags[p.workers + 1] = 0u;
    }
  }
}

}  // namespace ts
}  // namespace flute_dev
