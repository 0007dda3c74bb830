// flute-b200 — the LUT-dequant Stream-K GEMM kernel for the memory-bound regime
// (M <= 32 rows per launch), sm_100a.  Host launcher: qgemm_mma.cu.
//
// Reference semantics: flutesim::execute (engine.cpp:345) — Y = X * W_hat with
// W_hat = f16(scale * T[index]) (vec_lut.cpp:39-48) and fp32 accumulation;
// Stream-K ranges [floor(w*U/P), floor((w+1)*U/P)) over 128-deep units
// (n-tile major, k inner; streamk.cpp:17-58) with a fixed-order fixup of split
// tiles (engine.cpp:279-333).
//
// One CTA = one Stream-K worker = CW consumer warps (quartets taking stages
// round-robin; CW = 4 or 8, see launch_bits) + 1 producer warp + 1 epilogue
// warp, synchronised through mbarriers only (no CTA barrier in the steady
// state).  Every role walks the CTA's range the same way: tiles
// (segments) in descending order, and inside a tile stages of UPS units from
// the top k-slice down, so only a segment's last stage can be short.
//  * Producer.  Per stage: one 1-D bulk copy (UBLKCP) of the weights (a stage
//    is contiguous in the device layout), one of the group scales, and one
//    3-D TMA box (UTMALDG, 128B swizzle) of the X slice.  The weight/scale
//    copies of the first S stages are issued before the programmatic-
//    dependent-launch wait, so they overlap the previous kernel in the stream
//    (OCC = 2 configurations leave room for that CTA to be co-resident).
//  * Consumer warp q of a quartet owns k-steps 2q, 2q+1 of every unit of the
//    quartet's stages: LDS of its packed
//    pair indices, PRMT -> LDS from the 32-way duplicated vLUT, HMUL2 by the
//    group scale (operand-selector broadcast), mma.sync m16n8k16 with W^T as
//    the A operand (HMMA.16816.F32), X^T fragments via ldmatrix.  At the end
//    of a segment it parks its fp32 partial in shared memory and goes on.
//  * Epilogue warp.  Sums the CW warp partials in fixed order (deterministic),
//    then reduces split tiles off the critical path — cluster split-K through
//    DSMEM, or Stream-K: contributors publish bit-inverted fp32 partials (an
//    all-zero slot reads "not written"), finishers poll the data, add
//    contributors in ascending worker (= ascending k) order to their own
//    partial, write Y and re-zero the slots (graph / back-to-back safe).  The descending walk processes a split tile's contributor segment
//    first, so finishers rarely wait.
#pragma once

#include <cuda.h>
#include <cuda_fp16.h>

#include <type_traits>

#include "dequant.cuh"
#include "ptx.cuh"

namespace flute_dev {

// CW consumer warps (8 or 16; quartets of 4 warps take stages round-robin),
// then one producer warp and one epilogue warp.
constexpr int threads_for(int cw) { return 32 * (cw + 2); }
constexpr int kMaxStages = 16;
constexpr int kUnitN = 64;   // == flutesim::kUnitN (pack.hpp)
constexpr int kUnitK = 128;  // == flutesim::kUnitK: one Stream-K unit

constexpr int kMaxPeers = 8;

struct KParams {
  const uint8_t* w;
  const uint8_t* sc;
  const uint32_t* vlut;
  // Output: every value is stored to y_out[0..n_out) at [row * ldy + ycol0 + col].
  // n_out = 1, ldy = n, ycol0 = 0 is the plain GEMM; n_out > 1 with peer
  // pointers is the N-sharded layer's all-gather fused into the epilogue (each
  // rank writes its column slice straight into every rank's full Y).
  __half* y_out[kMaxPeers];
  int n_out, ldy, ycol0;
  float* slots;
  uint32_t* flags;
  int m, n;
  int tiles_k;      // units per 64-column tile
  int group_shift;  // log2(group size)
  int gp;           // padded groups per column
  int units;        // total units
  int workers;
  int stages;
  int use_ticket;
  int x3d;   // X tensor map is the 3-D {64, m, k/64} view (k % 64 == 0)
  // shared-memory plan (host: plan_smem in qgemm_mma.cu), byte offsets
  uint32_t part_off;      // partial rows that do not fit in the vLUT row gaps
  uint32_t part_stride;   // (unused by the device; kept for the host plan)
  uint32_t stage_off;     // first stage (1024-aligned)
  uint32_t stage_bytes;   // stage stride (multiple of 1024): [X | W | scales]
  uint32_t x_bytes;       // X region of a stage (1024-aligned; last 128 B = zero row)
  uint32_t bar_off;
  // Cluster split-K mode (cluster > 1): cluster c = 64-column tile c, its
  // `cluster` CTAs split the tile's k-units evenly and reduce through
  // distributed shared memory into rank 0 (receive buffer at recv_off).
  int cluster;
  uint32_t recv_off;
  int diag;  // FLUTE_DIAG bits (diag build only; results are wrong when set):
             // 1 skip dequant/MMA, 2 skip weight loads, 4 skip X, 8 skip scales,
             // 16 skip the Stream-K fixup, 32 skip the vLUT fill, 64 skip Y,
             // 128 skip the stage walk (no stage waits or copies), 256 no PDL
             // wait in the epilogue, 512 no cluster barriers, 1024 no PDL
             // wait in the producer
  unsigned long long* dbg;  // per-CTA timeline (diag build, FLUTE_DEBUG_TIMES)
};

template <int BITS, int BM, int UPS, int CW = 8>
struct Cfg {
  static constexpr int kConsumerWarps = CW;
  static constexpr int kGroups = CW / 4;  // quartets
  // shared-memory table rows: W2/W3 replicate their 16/64 entries to 256 so
  // index bytes need no masking (dequant.cuh), except at BM = 32, where the
  // 48-60 KB it would add leave too few pipeline stages (indices are masked)
  static constexpr int kEntries = BITS != 4 && BM == 32 ? 1 << (2 * BITS) : kTableRows<BITS>;
  static constexpr uint32_t kIndexMask = kEntries == 256 ? 0xFFFFFFFFu : BITS == 3 ? 0x3F3F3F3Fu : 0x0F0F0F0Fu;
  static constexpr int kLutBytes = kEntries * kLutRowBytes;
  static constexpr int kSubBytes = BITS * 1024;  // 64 x 128 weights
  static constexpr int kWBytes = UPS * kSubBytes;
  static constexpr int kFrag = (BM / 8) * 16;  // accumulator floats / lane
  static constexpr int kPartRows = kConsumerWarps * kFrag;
  // The vLUT uses the low 128 bytes of each 256-byte row (lane copies); the
  // first kPartRowsInLut partial-sum rows live in the high halves (a whole
  // number of warps' rows), the rest in a separate 128-byte-row buffer.
  static constexpr int kPartRowsInLut =
      (kPartRows < kEntries ? kPartRows : kEntries) / kFrag * kFrag;
  static constexpr int kPartBytes = (kPartRows - kPartRowsInLut) * 128;
  static constexpr int kBarBytes = 8 * (2 * kMaxStages + 2) + 64;
  // shared address (before + lane*4) of partial row r (part = separate buffer)
  static __device__ __forceinline__ uint32_t part_row(uint32_t lut, uint32_t part, int r) {
    return r < kPartRowsInLut ? lut + r * kLutRowBytes + kLutRowBytes / 2
                              : part + (r - kPartRowsInLut) * 128;
  }
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// Diagnostics (timeline stamps, FLUTE_DIAG bits) exist only in builds with
// -DFLUTE_DIAGNOSTICS (make diag); the product build compiles them out.
#ifndef FLUTE_SLEEP_PRODUCER
#define FLUTE_SLEEP_PRODUCER 1
#endif
#ifdef FLUTE_DIAGNOSTICS
#define FLUTE_STAMP(slot)                                                     \
  do {                                                                        \
    if (p.dbg) p.dbg[static_cast<size_t>(blockIdx.x) * 16 + (slot)] = gtimer(); \
  } while (0)
#define FLUTE_DIAG(bit) ((p.diag & (bit)) != 0)
#else
#define FLUTE_STAMP(slot) \
  do {                    \
  } while (0)
#define FLUTE_DIAG(bit) false
#endif

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

// The CTA's range [ubeg, uend) as segments (one per tile, descending); a
// segment covers k-slices [kt_bot, kt_top] of tile t.
struct SegRange {
  int t_hi, t_lo, ubeg, uend, tiles_k;
  __device__ __forceinline__ void init(int ub, int ue, int tk) {
    ubeg = ub;
    uend = ue;
    tiles_k = tk;
    t_hi = (ue - 1) / tk;
    t_lo = ub / tk;
  }
  __device__ __forceinline__ int top(int t) const {
    return t == t_hi ? uend - 1 - t * tiles_k : tiles_k - 1;
  }
  __device__ __forceinline__ int bot(int t) const { return t == t_lo ? ubeg - t * tiles_k : 0; }
};

// Stage ring position (slot s, phase parity ph).
struct Ring {
  int s = 0;
  uint32_t ph = 0;
  __device__ __forceinline__ void advance(int S) {
    if (++s == S) {
      s = 0;
      ph ^= 1u;
    }
  }
};

// OCC = CTAs per SM the register budget is sized for.  OCC = 2 lets a CTA of
// the NEXT launch (programmatic dependent launch) co-reside with this one, so
// its prologue and weight prefetch overlap this launch's tail; the host keeps
// shared memory within half an SM for those configurations.
template <int BITS, int BM, int UPS, int OCC, int CW>
__global__ void __launch_bounds__(threads_for(CW), OCC)
    qgemm_mma_kernel(const __grid_constant__ CUtensorMap tmap_x, const KParams p) {
  using C = Cfg<BITS, BM, UPS, CW>;
  constexpr int kConsumerWarps = CW;
  constexpr int kProducerWarp = CW;
  constexpr int kEpilogueWarp = CW + 1;
  constexpr int MT = BM / 8;
  extern __shared__ __align__(1024) uint8_t smem[];

  const int S = p.stages;
  const uint32_t base = smem_u32(smem);
  const uint32_t lut = base;
  const uint32_t stages0 = base + p.stage_off;
  const uint32_t SB = p.stage_bytes;
  const uint32_t XB = p.x_bytes;
  // stage s: X at stages0 + s*SB, weights at +XB, scales at +XB+kWBytes
  auto xs_of = [&](int st) { return stages0 + st * SB; };
  auto ws_of = [&](int st) { return stages0 + st * SB + XB; };
  auto ss_of = [&](int st) { return stages0 + st * SB + XB + C::kWBytes; };
  const uint32_t part = base + p.part_off;  // partial rows >= kPartRowsInLut
  const uint32_t bars = base + p.bar_off;
  auto full = [&](int s) { return bars + 8 * s; };
  auto empty = [&](int s) { return bars + 8 * (kMaxStages + s); };
  const uint32_t epi_full = bars + 8 * (2 * kMaxStages);
  const uint32_t epi_empty = epi_full + 8;
  const uint32_t recv_bar = epi_empty + 8;
  uint32_t* misc = reinterpret_cast<uint32_t*>(smem + (recv_bar + 8 - base));

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    FLUTE_STAMP(0);
#ifdef FLUTE_DIAGNOSTICS
    if (p.dbg) {  // slot 13: the SM this CTA runs on
      uint32_t smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      p.dbg[static_cast<size_t>(blockIdx.x) * 16 + 13] = smid;
    }
#endif
    for (int s = 0; s < S; ++s) {
      mbar_init(full(s), 1);
      mbar_init(empty(s), 4);  // one arrive per warp of the stage's quartet
    }
    // every lane arrives on the partial-sum hand-off barriers (once per
    // segment): each lane's own shared stores / loads are then ordered by its
    // own release / the waiter's acquire
    mbar_init(epi_full, kConsumerWarps * 32);
    mbar_init(epi_empty, 32);
    if (p.cluster > 1) mbar_init(recv_bar, 32 * (p.cluster - 1));  // every sender lane arrives
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
  if (threadIdx.x == 0) FLUTE_STAMP(8);
  // cluster mode: the receive barrier must be initialised before any peer
  // arrives on it (waited for just before the first remote access)
  // Cluster phase 1 (every thread arrives here): barriers initialised.  Phase 2
  // (every thread arrives when it no longer needs a peer's shared memory,
  // every thread waits just before exit): no CTA exits while a peer may still
  // write its receive buffer — the DSMEM lifetime rule, at the cost of rank
  // > 0 outliving only rank 0's read of the buffer, not its whole epilogue.
  bool cl_arrived = false;
  if (p.cluster > 1 && !FLUTE_DIAG(512)) cluster_arrive_relaxed();
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
  SegRange R;
  R.init(ubeg, uend, tiles_k);

  if (warp == kProducerWarp) {
    // ===================== producer =====================
    // The whole warp walks the stages (uniform control flow keeps addresses in
    // uniform registers); one elected lane issues each copy.
    if (uend > ubeg && !FLUTE_DIAG(128)) {
      const bool leader = elect_one();
      if (leader) prefetch_tmap(&tmap_x);
      const uint64_t pol = policy_evict_first();
      if (lane == 0) FLUTE_STAMP(9);
      const bool do_w = !FLUTE_DIAG(2), do_x = !FLUTE_DIAG(4), do_s = !FLUTE_DIAG(8);
      // stage = units [t*tiles_k + lo, t*tiles_k + lo + ns) of tile t
      auto issue_ws = [&](int t, int lo, int ns, int s) {
        const int glo = (lo * kUnitK) >> gshift;
        const int ng = ((((lo + ns) * kUnitK) - 1) >> gshift) - glo + 1;
        const uint32_t xb = do_x ? (p.x3d ? 2 * UPS : 2 * ns) * p.m * 128 : 0;
        const uint32_t wb = do_w ? ns * C::kSubBytes : 0;
        const uint32_t sb = do_s ? ng * 128 : 0;
        if (leader) {
          mbar_arrive_expect_tx(full(s), xb + wb + sb);
          if (wb)
            bulk_g2s_hint(ws_of(s), p.w + static_cast<size_t>(t * tiles_k + lo) * C::kSubBytes,
                          wb, full(s), pol);
          if (sb)
            bulk_g2s(ss_of(s), p.sc + (static_cast<size_t>(t) * p.gp + glo) * 128, sb, full(s));
        }
      };
      auto issue_x = [&](int lo, int ns, int s) {
        if (!do_x || !leader) return;
        if (p.x3d) {
          tma_3d_g2s(xs_of(s), &tmap_x, 0, 0, lo * 2, full(s));
        } else {
          for (int c = 0; c < 2 * ns; ++c)
            tma_2d_g2s(xs_of(s) + c * p.m * 128, &tmap_x, lo * kUnitK + 64 * c, 0, full(s));
        }
      };
      // pass 1 (before the PDL wait): weights + scales of the first S stages
      int pre = 0;
      for (int t = R.t_hi; t >= R.t_lo && pre < S; --t) {
        const int bot = R.bot(t);
        for (int kt = R.top(t); kt >= bot && pre < S; kt -= UPS) {
          const int lo = kt - UPS + 1 > bot ? kt - UPS + 1 : bot;
          issue_ws(t, lo, kt - lo + 1, pre);
          ++pre;
        }
      }
      FLUTE_STAMP(1);
      if (!p.use_ticket && !FLUTE_DIAG(1024)) pdl_wait();  // X and the workspace belong to the previous kernel
      if (lane == 0) FLUTE_STAMP(10);
      Ring ring;
      int it = 0;
      for (int t = R.t_hi; t >= R.t_lo; --t) {
        const int bot = R.bot(t);
        for (int kt = R.top(t); kt >= bot; kt -= UPS, ++it) {
          const int lo = kt - UPS + 1 > bot ? kt - UPS + 1 : bot;
          if (it >= pre) {
            if (FLUTE_SLEEP_PRODUCER) mbar_wait_sleep(empty(ring.s), ring.ph ^ 1u);
            else mbar_wait(empty(ring.s), ring.ph ^ 1u);
            issue_ws(t, lo, kt - lo + 1, ring.s);
          }
          issue_x(lo, kt - lo + 1, ring.s);
          ring.advance(S);
        }
      }
    }
  } else if (warp == kEpilogueWarp) {
    // ===================== epilogue =====================
    if (!p.use_ticket && !FLUTE_DIAG(256)) pdl_wait();  // the workspace and Y belong to the previous kernel
    if (lane == 0) FLUTE_STAMP(12);
    int seg = 0;
    for (int tile = R.t_hi; uend > ubeg && tile >= R.t_lo; --tile, ++seg) {
      // fixed-order sum of the 8 warp partials, then free the buffer
      mbar_wait_sleep(epi_full, seg & 1);
      float accf[C::kFrag];
#pragma unroll
      for (int i = 0; i < C::kFrag; ++i) {
        float v;
        asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(C::part_row(lut, part, i) + lane * 4u));
        accf[i] = v;
      }
#pragma unroll
      for (int w = 1; w < kConsumerWarps; ++w) {
#pragma unroll
        for (int i = 0; i < C::kFrag; ++i) {
          float v;
          asm volatile("ld.shared.f32 %0, [%1];"
                       : "=f"(v)
                       : "r"(C::part_row(lut, part, w * C::kFrag + i) + lane * 4u));
          accf[i] += v;
        }
      }
      __syncwarp();
      mbar_arrive(epi_empty);

      if (lane == 0) FLUTE_STAMP(tile == R.t_lo ? 5 : 4);
      const int t0 = tile * tiles_k;
      const bool started = ubeg <= t0;
      const bool finished = uend >= t0 + tiles_k;
      if (FLUTE_DIAG(16) || FLUTE_DIAG(512)) goto write_y;
      if (p.cluster > 1) {
        // ---- cluster split-K: ranks > 0 push their partial into rank 0's
        // receive buffer through DSMEM; rank 0 adds them in rank order ----
        const uint32_t recv = base + p.recv_off;
        cluster_wait();  // every CTA has initialised its barriers
        if (crank != 0) {
          const uint32_t dst = mapa_shared(recv + (crank - 1) * C::kFrag * 128 + lane * 4, 0);
#pragma unroll
          for (int i = 0; i < C::kFrag; ++i) st_cluster_f32(dst + i * 128, accf[i]);
          mbar_arrive_remote(mapa_shared(recv_bar, 0));
          asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");  // phase 2
          cl_arrived = true;
          continue;
        }
        mbar_wait_cluster(recv_bar, 0);
        for (int r = 1; r < p.cluster; ++r) {
#pragma unroll
          for (int i = 0; i < C::kFrag; ++i) {
            float v;
            asm volatile("ld.shared.f32 %0, [%1];"
                         : "=f"(v)
                         : "r"(recv + ((r - 1) * C::kFrag + i) * 128 + lane * 4));
            accf[i] += v;
          }
        }
        asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");  // phase 2: buffer read
        cl_arrived = true;
        goto write_y;
      }
      if (!finished) {
        // contributor: publish the fp32 partial as bit-inverted words, so an
        // all-zero slot means "not written yet" (0xFFFFFFFF is never produced:
        // NaNs are canonicalised to 0x7FFFFFFF).  No flag, no fence: the
        // finisher polls the data itself.
        // (volatile = relaxed, system scope: straight to L2, immediate offsets)
        volatile uint32_t* my_slot =
            reinterpret_cast<volatile uint32_t*>(p.slots) + static_cast<size_t>(wid) * C::kFrag * 32 + lane;
#pragma unroll
        for (int i = 0; i < C::kFrag; ++i) {
          uint32_t b = __float_as_uint(accf[i]);
          if (b == 0xFFFFFFFFu) b = 0x7FFFFFFFu;
          my_slot[i * 32] = ~b;
        }
        continue;
      }
      if (!started) {
        // finisher: contributors = non-empty workers in [owner(t0), wid), added
        // to the own partial in ascending worker (= ascending k) order:
        // ((own + c_first) + c_next) + ...  — a fixed order, so results are
        // bitwise reproducible for a given worker count.
        const int first = owner_of(t0, U, P);
        for (int c = first; c < wid; ++c) {
          if (range_lo(c + 1, U, P) <= range_lo(c, U, P)) continue;
          volatile uint32_t* src =
              reinterpret_cast<volatile uint32_t*>(p.slots) + static_cast<size_t>(c) * C::kFrag * 32 + lane;
          // poll in chunks of 16 words (bounded registers), all loads of a
          // chunk in flight together
#pragma unroll
          for (int i0 = 0; i0 < C::kFrag; i0 += 16) {
            uint32_t v[16];
            bool ready;
            do {
              ready = true;
#pragma unroll
              for (int i = 0; i < 16; ++i) {
                v[i] = src[(i0 + i) * 32];
                ready &= v[i] != 0u;
              }
            } while (!ready);
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              accf[i0 + i] += __uint_as_float(~v[i]);
              src[(i0 + i) * 32] = 0u;  // re-arm (graph / back-to-back safe)
            }
          }
        }
        if (lane == 0) FLUTE_STAMP(7);
      }
    write_y:
      if (FLUTE_DIAG(64)) continue;
      // write Y (f16, RNE); accf[(mt*4 + j)*4 + r] is C[n][m] of atom j, m-tile mt
      const int g = lane >> 2, t = lane & 3;
      const int ncol0 = tile * kUnitN;
      // one copy of the store code per output buffer (the peer loop stays
      // rolled: unrolling it inside the fragment loops quadruples the kernel)
#pragma unroll 1
      for (int d = 0; d < p.n_out; ++d) {
        __half* yb = p.y_out[d] + p.ycol0;
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
          for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int r = 0; r < 4; ++r) {
              const int row = mt * 8 + 2 * t + (r & 1);
              const int col = ncol0 + 16 * j + g + 8 * (r >> 1);
              if (row < p.m && col < p.n)
                yb[static_cast<size_t>(row) * p.ldy + col] = __float2half_rn(accf[(mt * 4 + j) * 4 + r]);
            }
      }
    }
    if (lane == 0) FLUTE_STAMP(15);  // epilogue done (diag build)
  } else {
    // ===================== consumers =====================
    if (!FLUTE_DIAG(32)) fill_lut<BITS, kConsumerWarps * 32, C::kEntries>(lut, p.vlut, threadIdx.x);
    if (threadIdx.x == 0) FLUTE_STAMP(11);
    const uint32_t lane4 = static_cast<uint32_t>(lane) * 4u;
    // Quartets of 4 warps take stages round-robin (quartet h: stages i with
    // i % kGroups == h), so the warps sharing an SMSP are out of phase (one in
    // its LUT-lookup phase while another issues MMAs).  Warp q of a quartet
    // owns k-steps 2q and 2q+1 (16 deep each) of every unit of its stages.
    const int half = warp >> 2;  // this warp's quartet
    const int q4 = warp & 3;
    constexpr int KS = 2;  // k-steps per warp per unit
    // X stage = TMA box {64 k, m rows, 2*UPS chunks}, compact ([chunk][m][128 B],
    // 128B-swizzled by box row Rw = chunk*m + row).  ldmatrix lanes whose row is
    // >= m read the X region's last 128 bytes, which TMA never writes when
    // m < BM and which are zeroed here — so no zero-fill bytes move.
    // MT == 1: one ldmatrix.x4 per unit covers both k-steps (b0, b1 of each);
    // MT >= 2: per k-step, one ldmatrix.x4 per pair of m-tiles.
    constexpr int XL = MT == 1 ? 1 : KS * (MT / 2);
    uint32_t xoff[UPS][XL];
    {
      const int mrows = p.m;
      const int mat = lane >> 3;
#pragma unroll
      for (int xl = 0; xl < XL; ++xl) {
        int row, ks, colh;
        if (MT == 1) {
          ks = mat >> 1;
          colh = mat & 1;
          row = lane & 7;
        } else {
          constexpr int MH = MT / 2 > 0 ? MT / 2 : 1;
          ks = xl / MH;
          const int qq = xl % MH;
          colh = mat & 1;
          row = qq * 16 + (mat >> 1) * 8 + (lane & 7);
        }
        const int kstep = 2 * q4 + ks;
        const int col = (kstep & 3) * 2 + colh;
#pragma unroll
        for (int r = 0; r < UPS; ++r) {
          const int Rw = (2 * r + (kstep >> 2)) * mrows + row;
          xoff[r][xl] = row < mrows ? static_cast<uint32_t>(Rw * 128 + ((col ^ (Rw & 7)) << 4))
                                    : XB - 128u;
        }
      }
      if (mrows < BM) {
        for (int i = threadIdx.x; i < S * 8; i += kConsumerWarps * 32)
          asm volatile("st.shared.v4.u32 [%0], {%1, %1, %1, %1};" ::"r"(
                           xs_of(i >> 3) + XB - 128 + (i & 7) * 16),
                       "r"(0u));
      }
    }
    named_bar_sync(1, kConsumerWarps * 32);  // LUT + zero rows visible
    if (threadIdx.x == 0) FLUTE_STAMP(2);

    // this lane's bytes within a unit for k-step ks: W4 16 B at slot*16; W2
    // 8 B at slot*8; W3 8 B (lane words A, B) at slot*8 + 4 B (word C) at
    // 2048 + slot*4, slot = kstep*32 + lane
    const int slot0 = 2 * q4 * 32 + lane;
    const uint32_t w_lane = slot0 * (BITS == 4 ? 16 : 8);
    constexpr uint32_t kSlotStride = 32 * (BITS == 4 ? 16 : 8);  // next k-step
    const uint32_t s_lane = (lane >> 2) * 16;
    const int kw = 32 * q4;  // k offset of this warp's first k-step in a unit

    float acc[MT][4][4];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int r = 0; r < 4; ++r) acc[mt][j][r] = 0.f;
    Ring ring;  // position of the global stage counter
#ifdef FLUTE_DIAGNOSTICS
    // per-stage trace of consumer warp 0: {wait begin, data ready, compute done}
    int stage_no = 0;
    unsigned long long* trace =
        (p.dbg && threadIdx.x == 0)
            ? p.dbg + static_cast<size_t>(gridDim.x) * 16 + static_cast<size_t>(blockIdx.x) * 64 * 3
            : nullptr;
#endif

    // One stage of NS units [lo, lo + NS) in ring slot (s, ph).
    auto run_stage = [&](auto ns_tag, int lo, int s, uint32_t ph) {
      constexpr int NS = decltype(ns_tag)::value;
      if (FLUTE_DIAG(128)) return;
#ifdef FLUTE_DIAGNOSTICS
      if (trace && stage_no < 64) trace[stage_no * 3] = gtimer();
#endif
      mbar_wait(full(s), ph);
#ifdef FLUTE_DIAGNOSTICS
      if (trace && stage_no < 64) trace[stage_no * 3 + 1] = gtimer();
#endif
      const uint32_t wst = ws_of(s) + w_lane;
      const uint32_t sst = ss_of(s) + s_lane;
      const uint32_t xst = xs_of(s);
      const int glo = (lo * kUnitK) >> gshift;
      LaneBits<BITS> lb[NS][KS];
      uint4 sq[NS];
      uint32_t bf[NS][KS][MT][2];
#pragma unroll
      for (int r = 0; r < NS; ++r) {
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
          const uint32_t wr = wst + r * C::kSubBytes + ks * kSlotStride;
          if constexpr (BITS == 4) {
            lb[r][ks].w = lds128(wr);
          } else if constexpr (BITS == 2) {
            lb[r][ks].w = lds64(wr);
          } else {
            lb[r][ks].hi = lds64(wr);
            lb[r][ks].lo = lds32(ws_of(s) + r * C::kSubBytes + 2048 + (slot0 + 32 * ks) * 4);
          }
        }
        // both k-steps (32 k) share one group (group >= 32)
        const int gl = ((((lo + r) << 7) + kw) >> gshift) - glo;
        sq[r] = lds128(sst + gl * 128);
        if constexpr (MT == 1) {
          ldsm_x4(xst + xoff[r][0], bf[r][0][0][0], bf[r][0][0][1], bf[r][1][0][0], bf[r][1][0][1]);
        } else {
#pragma unroll
          for (int ks = 0; ks < KS; ++ks)
#pragma unroll
            for (int qq = 0; qq < MT / 2; ++qq)
              ldsm_x4(xst + xoff[r][ks * (MT / 2) + qq], bf[r][ks][2 * qq][0], bf[r][ks][2 * qq][1],
                      bf[r][ks][2 * qq + 1][0], bf[r][ks][2 * qq + 1][1]);
        }
      }
      // One arrive per warp: lane 0's release covers the warp's loads (same
      // instructions, all lanes).
      __syncwarp();
      if (lane == 0) mbar_arrive(empty(s));
      if (FLUTE_DIAG(1)) return;
#pragma unroll
      for (int r = 0; r < NS; ++r) {
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
          // all 16 lookups of the k-step first, then scale + MMA per atom
          uint32_t v[4][4];
#pragma unroll
          for (int j = 0; j < 4; ++j)
            lut_lookup4(atom_index_bytes<BITS>(lb[r][ks], j) & C::kIndexMask, lane4, lut, v[j]);
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const uint32_t scw = j == 0 ? sq[r].x : j == 1 ? sq[r].y : j == 2 ? sq[r].z : sq[r].w;
            uint32_t a[4];
            lut_scale4(v[j], scw, a);
#pragma unroll
            for (int mt = 0; mt < MT; ++mt)
              mma_16816(acc[mt][j], a, bf[r][ks][mt][0], bf[r][ks][mt][1]);
          }
        }
      }
#ifdef FLUTE_DIAGNOSTICS
      if (trace && stage_no < 64) {
        float sink = 0.f;  // make the stamp wait for this warp's MMAs to retire
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) sink += acc[mt][0][0] + acc[mt][3][3];
        trace[stage_no * 3 + 2] = gtimer() + (sink == 1.2345e-30f ? 1 : 0);
      }
      ++stage_no;
#endif
    };

    int seg = 0;
    int parity = 0;  // global stage counter % kGroups
    for (int tile = R.t_hi; uend > ubeg && tile >= R.t_lo; --tile, ++seg) {
      const int bot = R.bot(tile);
      int kt = R.top(tile);
      // full stages, then at most one short stage; this half takes every
      // other stage of the CTA-wide sequence
      for (; kt - bot + 1 >= UPS; kt -= UPS) {
        if (parity == half) run_stage(std::integral_constant<int, UPS>{}, kt - UPS + 1, ring.s, ring.ph);
        ring.advance(S);
        if (++parity == C::kGroups) parity = 0;
      }
      if constexpr (UPS > 1) {
        const int rem = kt - bot + 1;
        if (rem > 0) {
          if (parity == half) {
            if (rem == 1) {
              run_stage(std::integral_constant<int, 1>{}, bot, ring.s, ring.ph);
            } else if constexpr (UPS > 2) {
              if (rem == 2) {
                run_stage(std::integral_constant<int, 2>{}, bot, ring.s, ring.ph);
              } else if constexpr (UPS > 3) {
                if (rem == 3) run_stage(std::integral_constant<int, 3>{}, bot, ring.s, ring.ph);
              }
            }
          }
          ring.advance(S);
          if (++parity == C::kGroups) parity = 0;
        }
      }
      // ---- segment end: every warp parks its partial for the epilogue ----
      if (seg > 0) mbar_wait(epi_empty, (seg - 1) & 1);
      const float* accf = &acc[0][0][0];
      // this warp's rows are all in the vLUT gaps or all in the separate buffer
      const bool in_lut = warp * C::kFrag < C::kPartRowsInLut;
      const uint32_t row0 = (in_lut ? lut + warp * C::kFrag * kLutRowBytes + kLutRowBytes / 2
                                    : part + (warp * C::kFrag - C::kPartRowsInLut) * 128) +
                            lane * 4u;
      const uint32_t rstride = in_lut ? kLutRowBytes : 128u;
#pragma unroll
      for (int i = 0; i < C::kFrag; ++i)
        asm volatile("st.shared.f32 [%0], %1;" ::"r"(row0 + i * rstride), "f"(accf[i]));
      __syncwarp();
      mbar_arrive(epi_full);
#pragma unroll
      for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
          for (int r = 0; r < 4; ++r) acc[mt][j][r] = 0.f;
    }
  }

  if (threadIdx.x == 0) FLUTE_STAMP(6);
  // cluster phase 2 (see the top): threads that have not arrived yet wait
  // out phase 1 and arrive; then every thread waits for the whole cluster
  if (p.cluster > 1 && !FLUTE_DIAG(512)) {
    if (!cl_arrived) {
      cluster_wait();
      asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
    }
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
  }
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
