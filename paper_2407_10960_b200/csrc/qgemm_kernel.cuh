// flute-b200 — the LUT-dequant Stream-K GEMM kernel for the memory-bound regime
// (M <= 32 rows per launch), sm_100a.  Host launcher: qgemm_mma.cu.
//
// Reference semantics: flutesim::execute (engine.cpp:345) — Y = X * W_hat with
// W_hat = f16(scale * T[index]) (vec_lut.cpp:39-48) and fp32 accumulation;
// Stream-K ranges [floor(w*U/P), floor((w+1)*U/P)) over 128-deep sub-units
// (n-tile major, k inner; streamk.cpp:17-58) with a fixed-order fixup of split
// tiles (engine.cpp:279-333).
//
// One CTA = one Stream-K worker: 8 consumer warps + 1 producer warp.
//  * Stages.  The CTA walks its sub-units in descending order and groups up
//    to UPS consecutive sub-units of the same 64-column tile into one stage:
//    its weights and scales are contiguous in the device layout (one 1-D bulk
//    copy each, UBLKCP) and its X slice is one 3-D TMA box {64 k, BM rows,
//    2*UPS chunks}, 128B-swizzled (UTMALDG).  Three copies per stage keep the
//    single producer thread far ahead of HBM.  The weight/scale copies of the
//    first S stages are issued before the programmatic-dependent-launch wait,
//    so they overlap the previous kernel in the stream.
//  * Consumer warp w owns k-steps {w, w+8, ...} of a stage: LDS of its packed
//    pair indices, PRMT -> LDS from the 32-way duplicated vLUT, HMUL2 by the
//    group scale (operand-selector broadcast), mma.sync m16n8k16 with W^T as
//    the A operand (HMMA.16816.F32), X^T fragments via ldmatrix.
//  * Descending walk: a split tile's contributor segment (the range's tail) is
//    processed first and published early; the finisher segment (the range's
//    head) is reduced last, so the finisher rarely waits.
//  * Split tiles reduce through an fp32 workspace: contributors store their
//    partial and release-add the finisher's flag; the finisher acquires, sums
//    contributors in ascending worker (= ascending k) order, adds its own
//    partial, writes Y and re-arms its flag (graph / back-to-back safe).
#pragma once

#include <cuda.h>
#include <cuda_fp16.h>

#include <type_traits>

#include "dequant.cuh"
#include "ptx.cuh"

namespace flute_dev {

// Consumer warps per CTA: CW in {8, 16} (template); plus one producer warp.
template <int CW>
constexpr int threads_for() {
  return 32 * (CW + 1);
}
constexpr int kMaxStages = 16;
constexpr int kUnitN = 64;   // == flutesim::kUnitN (pack.hpp)
constexpr int kUnitK = 128;  // == flutesim::kUnitK: one Stream-K sub-unit

struct KParams {
  const uint8_t* w;
  const uint8_t* sc;
  const uint32_t* vlut;
  __half* y;
  float* slots;
  uint32_t* flags;
  int m, n;
  int tiles_k;      // sub-units per 64-column tile
  int group_shift;  // log2(group size)
  int gp;           // padded groups per column
  int units;        // total sub-units
  int workers;
  int stages;
  int use_ticket;
  int x3d;   // X tensor map is the 3-D {64, m, k/64} view (k % 64 == 0)
  int diag;  // FLUTE_DIAG bits (diagnostics; results are wrong when set):
             // 1 skip dequant/MMA, 2 skip weight loads, 4 skip X, 8 skip scales
  unsigned long long* dbg;  // optional per-CTA timeline (FLUTE_DEBUG_TIMES)
};

template <int BITS, int BM, int UPS, int CW>
struct Cfg {
  static constexpr int kLutBytes = (1 << (2 * BITS)) * kLutRowBytes;
  static constexpr int kSubBytes = BITS * 1024;             // 64 x 128 weights
  static constexpr int kChunks = 2 * UPS;                   // 64-wide k chunks of X
  static constexpr int kXBytes = kChunks * BM * 128;
  static constexpr int kWBytes = UPS * kSubBytes;
  static constexpr int kScBytes = UPS * 4 * 128;            // <= 4 groups per sub-unit
  static constexpr int kFrag = (BM / 8) * 16;               // accumulator floats / lane
  static constexpr int kRedBytes = (CW / 2) * kFrag * 32 * 4 + 128;  // + a zero row for ldmatrix
  static constexpr int kStageBytes = kXBytes + kWBytes + kScBytes;
  static constexpr size_t smem_bytes(int S) {
    return static_cast<size_t>(kLutBytes) + static_cast<size_t>(S) * kStageBytes + kRedBytes +
           2 * 8 * kMaxStages + 64;
  }
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define FLUTE_STAMP(slot)                                                     \
  do {                                                                        \
    if (p.dbg) p.dbg[static_cast<size_t>(blockIdx.x) * 8 + (slot)] = gtimer(); \
  } while (0)

// Host guarantees units * (workers + 1) < 2^31, so 32-bit math is exact.
__device__ __forceinline__ int range_lo(int w, int U, int P) {
  return static_cast<int>(static_cast<uint32_t>(U) * static_cast<uint32_t>(w) /
                          static_cast<uint32_t>(P));
}

__device__ __forceinline__ int owner_of(int x, int U, int P) {
  int w = static_cast<int>(static_cast<uint32_t>(x) * static_cast<uint32_t>(P) /
                           static_cast<uint32_t>(U));
  if (w >= P) w = P - 1;
  while (w + 1 < P && range_lo(w + 1, U, P) <= x) ++w;
  while (w > 0 && range_lo(w, U, P) > x) --w;
  return w;
}

// Descending walk over a CTA range in stages of <= UPS sub-units that never
// cross a tile boundary.  Producer and consumers run identical copies.
template <int UPS>
struct StageWalk {
  int hi, tile, kt;  // highest remaining sub-unit, its tile and k-slice
  int nsub, lo_kt;   // current stage: sub-units [hi-nsub+1, hi], k-slices [lo_kt, kt]
  __device__ __forceinline__ void init(int uend, int tiles_k) {
    hi = uend - 1;
    tile = hi / tiles_k;
    kt = hi - tile * tiles_k;
  }
  __device__ __forceinline__ void shape(int ubeg) {
    int n = kt + 1 < UPS ? kt + 1 : UPS;
    nsub = hi - ubeg + 1 < n ? hi - ubeg + 1 : n;
    lo_kt = kt - nsub + 1;
  }
  __device__ __forceinline__ void next(int tiles_k) {
    hi -= nsub;
    if (lo_kt == 0) {
      --tile;
      kt = tiles_k - 1;
    } else {
      kt = lo_kt - 1;
    }
  }
};

template <int BITS, int BM, int UPS, int CW>
__global__ void __launch_bounds__(threads_for<CW>(), 1)
    qgemm_mma_kernel(const __grid_constant__ CUtensorMap tmap_x, const KParams p) {
  using C = Cfg<BITS, BM, UPS, CW>;
  constexpr int kConsumerWarps = CW;
  constexpr int R = CW / 8;  // warps sharing one k-step: warp w takes sub-units r == w/8 (mod R)
  constexpr int MT = BM / 8;
  extern __shared__ __align__(1024) uint8_t smem[];

  const int S = p.stages;
  const uint32_t base = smem_u32(smem);
  const uint32_t lut = base;
  const uint32_t xs = base + C::kLutBytes;
  const uint32_t ws = xs + S * C::kXBytes;
  const uint32_t ss = ws + S * C::kWBytes;
  const uint32_t red = ss + S * C::kScBytes;
  const uint32_t bars = red + C::kRedBytes;  // full[kMaxStages], empty[kMaxStages]
  uint32_t* misc = reinterpret_cast<uint32_t*>(smem + (bars - base) + 16 * kMaxStages);
  auto full = [&](int s) { return bars + 8 * s; };
  auto empty = [&](int s) { return bars + 8 * (kMaxStages + s); };

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    FLUTE_STAMP(0);
    for (int s = 0; s < S; ++s) {
      mbar_init(full(s), 1);
      mbar_init(empty(s), kConsumerWarps);
    }
    fence_mbar_init();
  }
  int wid = blockIdx.x;
  if (p.use_ticket) {
    // More workers than co-resident CTAs: take worker ids in start order so a
    // finisher only ever waits on CTAs that are already running.
    pdl_wait();
    if (threadIdx.x == 0) misc[0] = atomicAdd(p.flags + p.workers, 1u);
  }
  __syncthreads();
  if (p.use_ticket) wid = static_cast<int>(misc[0]);
  pdl_launch_dependents();

  const int U = p.units;
  const int P = p.workers;
  const int ubeg = range_lo(wid, U, P);
  const int uend = range_lo(wid + 1, U, P);
  const int tiles_k = p.tiles_k;
  const int gshift = p.group_shift;

  if (warp == kConsumerWarps) {
    // ===================== producer =====================
    if (lane == 0 && uend > ubeg) {
      prefetch_tmap(&tmap_x);
      const uint64_t pol = policy_evict_first();
      const bool do_w = !(p.diag & 2), do_x = !(p.diag & 4), do_s = !(p.diag & 8);
      auto issue_ws = [&](const StageWalk<UPS>& sw, int s) {
        const int glo = (sw.lo_kt * kUnitK) >> gshift;
        const int ng = (((sw.kt + 1) * kUnitK - 1) >> gshift) - glo + 1;
        const uint32_t xb = do_x ? (p.x3d ? 2 * UPS : 2 * sw.nsub) * p.m * 128 : 0;
        const uint32_t wb = do_w ? sw.nsub * C::kSubBytes : 0;
        const uint32_t sb = do_s ? ng * 128 : 0;
        mbar_arrive_expect_tx(full(s), xb + wb + sb);
        if (wb)
          bulk_g2s_hint(ws + s * C::kWBytes,
                        p.w + static_cast<size_t>(sw.hi - sw.nsub + 1) * C::kSubBytes, wb, full(s),
                        pol);
        if (sb)
          bulk_g2s(ss + s * C::kScBytes, p.sc + (static_cast<size_t>(sw.tile) * p.gp + glo) * 128,
                   sb, full(s));
      };
      auto issue_x = [&](const StageWalk<UPS>& sw, int s) {
        if (!do_x) return;
        if (p.x3d) {
          tma_3d_g2s(xs + s * C::kXBytes, &tmap_x, 0, 0, sw.lo_kt * 2, full(s));
        } else {
          for (int c = 0; c < 2 * sw.nsub; ++c)
            tma_2d_g2s(xs + s * C::kXBytes + c * p.m * 128, &tmap_x, sw.lo_kt * kUnitK + 64 * c, 0,
                       full(s));
        }
      };
      // pass 1 (before the PDL wait): weights + scales of the first S stages
      StageWalk<UPS> w1;
      w1.init(uend, tiles_k);
      int pre = 0;
      while (pre < S && w1.hi >= ubeg) {
        w1.shape(ubeg);
        issue_ws(w1, pre);
        w1.next(tiles_k);
        ++pre;
      }
      FLUTE_STAMP(1);
      if (!p.use_ticket) pdl_wait();  // X and the workspace belong to the previous kernel
      StageWalk<UPS> w2;
      w2.init(uend, tiles_k);
      int s = 0;
      uint32_t ph = 0;
      for (int it = 0; w2.hi >= ubeg; ++it) {
        w2.shape(ubeg);
        if (it >= pre) {
          mbar_wait(empty(s), ph ^ 1u);
          issue_ws(w2, s);
        }
        issue_x(w2, s);
        w2.next(tiles_k);
        if (++s == S) {
          s = 0;
          ph ^= 1u;
        }
      }
    }
  } else {
    // ===================== consumers =====================
    fill_lut<BITS, kConsumerWarps * 32>(lut, p.vlut, threadIdx.x);
    if (!p.use_ticket) pdl_wait();
    named_bar_sync(1, kConsumerWarps * 32);
    if (threadIdx.x == 0) FLUTE_STAMP(2);

    const uint32_t lane4 = static_cast<uint32_t>(lane) * 4u;
    // X stage = TMA box {64 k, m rows, 2*UPS chunks}, compact ([chunk][m][128 B],
    // 128B-swizzled by box row R = chunk*m + row).  ldmatrix lanes whose row is
    // >= m read a shared zero row instead, so no zero-fill bytes move.
    const int mrows = p.m;
    int lrow[MT > 1 ? MT / 2 : 1];  // this lane's ldmatrix row per x4 (or x2)
    int lcol[MT > 1 ? MT / 2 : 1];  // its 16-byte column chunk within 128 B
    {
      const int c0 = ((warp & 7) & 3) * 2;
      if constexpr (MT == 1) {
        lrow[0] = lane & 7;
        lcol[0] = c0 + ((lane >> 3) & 1);
      } else {
#pragma unroll
        for (int q = 0; q < MT / 2; ++q) {
          const int mat = lane >> 3;
          lrow[q] = q * 16 + (mat >> 1) * 8 + (lane & 7);
          lcol[q] = c0 + (mat & 1);
        }
      }
    }
    const uint32_t zrow = red + C::kRedBytes - 128;  // never written by the reduction
    if (warp == 0) asm volatile("st.shared.v4.u32 [%0], {%1, %1, %1, %1};" ::"r"(zrow + lane * 16 % 128), "r"(0u));
    named_bar_sync(1, kConsumerWarps * 32);
    auto x_addr = [&](uint32_t xstage, int chunk, int q) -> uint32_t {
      const int row = lrow[q];
      if (row >= mrows) return zrow;
      const int R = chunk * mrows + row;
      return xstage + R * 128 + ((lcol[q] ^ (R & 7)) << 4);
    };

    float acc[MT][4][4];
    StageWalk<UPS> sw;
    sw.init(uend, tiles_k);
    int s = 0;
    uint32_t ph = 0;
    bool first_stage = true;
    for (; sw.hi >= ubeg; sw.next(tiles_k), s = (s + 1 == S) ? 0 : s + 1, ph ^= (s == 0) ? 1u : 0u) {
      sw.shape(ubeg);
      if (first_stage || sw.kt == tiles_k - 1) {
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
          for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int r = 0; r < 4; ++r) acc[mt][j][r] = 0.f;
      }
      mbar_wait(full(s), ph);
      if (first_stage && threadIdx.x == 0) FLUTE_STAMP(3);
      first_stage = false;

      // ---- stage -> registers (all loads first), then dequant + MMA ----
      // NS = sub-units in this stage; full stages (the common case) take the
      // NS = UPS instantiation, free of per-sub-unit predicates.
      const uint32_t wst = ws + s * C::kWBytes;
      const uint32_t sst = ss + s * C::kScBytes;
      const uint32_t xst = xs + s * C::kXBytes;
      const int glo = (sw.lo_kt * kUnitK) >> gshift;
      const int kstep = warp & 7;   // 16-deep k step within a sub-unit
      const int rsel = warp >> 3;   // this warp's sub-unit phase (0..R-1)
      auto run_stage = [&](auto ns_tag) {
        constexpr int NS = decltype(ns_tag)::value;
        constexpr int NR = (NS + R - 1) / R;  // sub-units per warp (upper bound)
        LaneBits<BITS> lb[NR];
        uint4 sq[NR];
        uint32_t bf[NR][MT][2];
        bool live[NR];
#pragma unroll
        for (int rr = 0; rr < NR; ++rr) {
          const int r = rr * R + rsel;
          live[rr] = (NS % R == 0) || r < NS;
          if (!live[rr]) continue;
          const uint32_t wr = wst + r * C::kSubBytes;
          const int lslot = kstep * 32 + lane;
          if constexpr (BITS == 4) {
            lb[rr].w = lds128(wr + lslot * 16);
          } else if constexpr (BITS == 2) {
            lb[rr].w = lds64(wr + lslot * 8);
          } else {
            lb[rr].hi = lds64(wr + lslot * 8);
            lb[rr].lo = lds32(wr + 2048 + lslot * 4);
          }
          const int gl = ((((sw.lo_kt + r) << 7) + 16 * kstep) >> gshift) - glo;
          sq[rr] = lds128(sst + gl * 128 + (lane >> 2) * 16);
          const int chunk = 2 * r + (kstep >> 2);
          if constexpr (MT == 1) {
            ldsm_x2(x_addr(xst, chunk, 0), bf[rr][0][0], bf[rr][0][1]);
          } else {
#pragma unroll
            for (int q = 0; q < MT / 2; ++q)
              ldsm_x4(x_addr(xst, chunk, q), bf[rr][2 * q][0], bf[rr][2 * q][1],
                      bf[rr][2 * q + 1][0], bf[rr][2 * q + 1][1]);
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(empty(s));
        if (p.diag & 1) return;
#pragma unroll
        for (int rr = 0; rr < NR; ++rr) {
          if (!live[rr]) continue;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const uint32_t scw =
                j == 0 ? sq[rr].x : j == 1 ? sq[rr].y : j == 2 ? sq[rr].z : sq[rr].w;
            uint32_t a[4];
            lut_dequant4(atom_index_bytes<BITS>(lb[rr], j), lane4, lut, scw, a);
#pragma unroll
            for (int mt = 0; mt < MT; ++mt) mma_16816(acc[mt][j], a, bf[rr][mt][0], bf[rr][mt][1]);
          }
        }
      };
      if (sw.nsub == UPS) {
        run_stage(std::integral_constant<int, UPS>{});
      } else if (sw.nsub == 1) {
        run_stage(std::integral_constant<int, 1>{});
      } else if constexpr (UPS > 2) {
        if (sw.nsub == 2) run_stage(std::integral_constant<int, 2>{});
        else run_stage(std::integral_constant<int, (UPS > 3 ? 3 : 1)>{});
      }

      const bool seg_end = sw.lo_kt == 0 || sw.hi - sw.nsub + 1 == ubeg;
      if (!seg_end) continue;

      // ---- segment end: deterministic CTA reduction (tree over warps) ----
      float* accf = &acc[0][0][0];
      auto red_addr = [&](int sl, int i) { return red + ((sl * C::kFrag + i) * 32 + lane) * 4u; };
#pragma unroll
      for (int half = CW / 2; half >= 1; half >>= 1) {
        if (warp >= half && warp < 2 * half) {
#pragma unroll
          for (int i = 0; i < C::kFrag; ++i)
            asm volatile("st.shared.f32 [%0], %1;" ::"r"(red_addr(warp - half, i)), "f"(accf[i]));
        }
        named_bar_sync(1, kConsumerWarps * 32);
        if (warp < half) {
#pragma unroll
          for (int i = 0; i < C::kFrag; ++i) {
            float v;
            asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(red_addr(warp, i)));
            accf[i] += v;
          }
        }
        named_bar_sync(1, kConsumerWarps * 32);
      }

      const int tile = sw.tile;
      const bool last_seg = sw.hi - sw.nsub + 1 == ubeg;
      if (threadIdx.x == 0) FLUTE_STAMP(last_seg ? 5 : 4);
      if (warp == 0) {
        const int t0 = tile * tiles_k;
        const bool started = ubeg <= t0;
        const bool finished = uend >= t0 + tiles_k;
        if (!finished) {
          // contributor: publish the fp32 partial, then release-add the
          // finisher's flag.
          float* my_slot = p.slots + static_cast<size_t>(wid) * C::kFrag * 32;
#pragma unroll
          for (int i = 0; i < C::kFrag; ++i) my_slot[i * 32 + lane] = accf[i];
          asm volatile("fence.acq_rel.gpu;" ::: "memory");
          __syncwarp();
          if (lane == 0) red_release_gpu_add(p.flags + owner_of(t0 + tiles_k - 1, U, P), 1u);
        } else {
          if (!started) {
            // finisher: contributors = non-empty workers in [owner(t0), wid)
            const int first = owner_of(t0, U, P);
            uint32_t expect = 0;
            for (int c = first; c < wid; ++c)
              expect += range_lo(c + 1, U, P) > range_lo(c, U, P) ? 1u : 0u;
            while (ld_acquire_gpu(p.flags + wid) < expect) {
            }
            if (threadIdx.x == 0) FLUTE_STAMP(7);
            // ((c_first + c_next) + ...) + own
            float sum[C::kFrag];
            bool have = false;
            for (int c = first; c < wid; ++c) {
              if (range_lo(c + 1, U, P) <= range_lo(c, U, P)) continue;
              const float* src = p.slots + static_cast<size_t>(c) * C::kFrag * 32 + lane;
              if (!have) {
#pragma unroll
                for (int i = 0; i < C::kFrag; ++i) sum[i] = __ldcg(src + i * 32);
              } else {
#pragma unroll
                for (int i = 0; i < C::kFrag; ++i) sum[i] += __ldcg(src + i * 32);
              }
              have = true;
            }
#pragma unroll
            for (int i = 0; i < C::kFrag; ++i) accf[i] = sum[i] + accf[i];
            __syncwarp();
            if (lane == 0) *reinterpret_cast<volatile uint32_t*>(p.flags + wid) = 0u;
          }
          // write Y (f16, RNE)
          const int g = lane >> 2, t = lane & 3;
          const int ncol0 = tile * kUnitN;
#pragma unroll
          for (int mt = 0; mt < MT; ++mt)
#pragma unroll
            for (int j = 0; j < 4; ++j)
#pragma unroll
              for (int r = 0; r < 4; ++r) {
                const int row = mt * 8 + 2 * t + (r & 1);
                const int col = ncol0 + 16 * j + g + 8 * (r >> 1);
                if (row < p.m && col < p.n)
                  p.y[static_cast<size_t>(row) * p.n + col] = __float2half_rn(acc[mt][j][r]);
              }
        }
      }
    }
  }

  if (threadIdx.x == 0) FLUTE_STAMP(6);
  if (p.use_ticket) {
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      const uint32_t done = atomicAdd(p.flags + p.workers + 1, 1u);
      if (done == static_cast<uint32_t>(P) - 1u) {
        p.flags[p.workers] = 0u;
        p.flags[p.workers + 1] = 0u;
      }
    }
  }
}

}  // namespace flute_dev
