// flute-b200 — the LUT-dequant Stream-K GEMM for the memory-bound regime
// (M <= 32 per launch), sm_100a.
//
// Reference semantics: flutesim::execute (engine.cpp:345) — Y = X * W_hat with
// W_hat = f16(scale * T[index]) and fp32 accumulation; Stream-K ranges
// [floor(w*U/P), floor((w+1)*U/P)) over units (n-tile major, k inner) with a
// fixed-order fixup of split tiles (streamk.cpp:17-58, engine.cpp:279-333).
//
// One CTA = one Stream-K worker, 8 consumer warps + 1 producer warp:
//  * producer (one lane): streams the CTA's units with 1-D bulk async copies
//    (weights, scales; UBLKCP) and 2-D TMA (the X slice, 128B-swizzled;
//    UTMALDG) into an S-stage shared-memory ring guarded by mbarriers.  The
//    weight/scale prefetch of the first S stages is issued before the
//    programmatic-dependent-launch wait, so it overlaps the previous kernel.
//  * consumer warp w owns k-step w (16 deep) of every 64x128 unit: one LDS of
//    its packed pair indices, PRMT -> LDS from the 32-way duplicated vLUT,
//    HMUL2 by the group scale, and mma.sync m16n8k16 with W^T as the A operand
//    (HMMA.16816.F32), X^T fragments via ldmatrix.
//  * a CTA walks its range in *descending* unit order, so the contributor
//    segment of a split tile (its range's tail) is published first and the
//    finisher segment (its range's head) is reduced last — the finisher never
//    stalls waiting for a neighbour that is still mid-range.
//  * split tiles reduce through an fp32 workspace: contributors store their
//    partial and release-add the finisher's flag; the finisher acquires,
//    sums contributors in ascending worker (= ascending k) order, adds its own
//    partial, writes Y, and re-zeroes its flag (graph/launch-safe).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <mutex>
#include <string>
#include <unordered_map>

#include "dequant.cuh"
#include "device_api.h"
#include "flutesim/errors.hpp"
#include "ptx.cuh"

namespace flute_dev {

constexpr int kConsumerWarps = 8;
constexpr int kThreads = 32 * (kConsumerWarps + 1);
constexpr int kMaxStages = 16;
constexpr int kUnitN = 64;   // == flutesim::kUnitN (pack.hpp)
constexpr int kUnitK = 128;  // == flutesim::kUnitK

struct KParams {
  const uint8_t* w;
  const uint8_t* sc;
  const uint32_t* vlut;
  __half* y;
  float* slots;
  uint32_t* flags;
  int m, n;
  int tiles_k;
  int group;
  int gp;  // padded groups per column
  long long units;
  int workers;
  int stages;
  int use_ticket;
};

template <int BITS, int BM>
struct Cfg {
  static constexpr int kLutBytes = (1 << (2 * BITS)) * kLutRowBytes;
  static constexpr int kUnitBytes = BITS * 1024;  // 64 x 128 weights
  static constexpr int kXBytes = 2 * BM * 128;    // two 64-wide TMA boxes
  static constexpr int kScBytes = 512;            // <= 4 groups x 64 scales
  static constexpr int kFrag = (BM / 8) * 16;     // accumulator floats / lane
  static constexpr int kRedBytes = 4 * kFrag * 32 * 4;
  static constexpr int kStageBytes = kXBytes + kUnitBytes + kScBytes;
  static size_t smem_bytes(int S) {
    return static_cast<size_t>(kLutBytes) + static_cast<size_t>(S) * kStageBytes + kRedBytes +
           2 * 8 * kMaxStages + 64;
  }
};

__device__ __forceinline__ long long range_lo(long long w, long long U, long long P) {
  return U * w / P;
}

__device__ __forceinline__ int owner_of(long long x, long long U, int P) {
  int w = static_cast<int>((x * P) / U);
  if (w >= P) w = P - 1;
  while (w + 1 < P && range_lo(w + 1, U, P) <= x) ++w;
  while (w > 0 && range_lo(w, U, P) > x) --w;
  return w;
}

template <int BITS, int BM>
__global__ void __launch_bounds__(kThreads, 1)
    qgemm_mma_kernel(const __grid_constant__ CUtensorMap tmap_x, const KParams p) {
  using C = Cfg<BITS, BM>;
  constexpr int MT = BM / 8;
  extern __shared__ __align__(1024) uint8_t smem[];

  const int S = p.stages;
  const uint32_t base = smem_u32(smem);
  const uint32_t lut = base;
  const uint32_t xs = base + C::kLutBytes;
  const uint32_t ws = xs + S * C::kXBytes;
  const uint32_t ss = ws + S * C::kUnitBytes;
  const uint32_t red = ss + S * C::kScBytes;
  const uint32_t bars = red + C::kRedBytes;  // full[kMaxStages], empty[kMaxStages]
  uint32_t* misc = reinterpret_cast<uint32_t*>(smem + (bars - base) + 16 * kMaxStages);
  auto full = [&](int s) { return bars + 8 * s; };
  auto empty = [&](int s) { return bars + 8 * (kMaxStages + s); };

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
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

  const long long U = p.units;
  const int P = p.workers;
  const long long ubeg = range_lo(wid, U, P);
  const long long uend = range_lo(wid + 1, U, P);
  const int nunits = static_cast<int>(uend - ubeg);
  const int tiles_k = p.tiles_k;
  const int group = p.group;
  const int ng = group >= kUnitK ? 1 : kUnitK / group;

  if (warp == kConsumerWarps) {
    // ===================== producer =====================
    if (lane == 0 && nunits > 0) {
      prefetch_tmap(&tmap_x);
      const uint64_t pol = policy_evict_first();
      const uint32_t stage_tx = C::kXBytes + C::kUnitBytes + ng * 128;
      auto issue_ws = [&](int it) {
        const int s = it % S;
        const long long u = uend - 1 - it;
        const long long nt = u / tiles_k;
        const int kt = static_cast<int>(u % tiles_k);
        const long long glo = static_cast<long long>(kt) * kUnitK / group;
        mbar_arrive_expect_tx(full(s), stage_tx);
        bulk_g2s_hint(ws + s * C::kUnitBytes, p.w + u * C::kUnitBytes, C::kUnitBytes, full(s), pol);
        bulk_g2s(ss + s * C::kScBytes, p.sc + (nt * p.gp + glo) * 128, ng * 128, full(s));
      };
      auto issue_x = [&](int it) {
        const int s = it % S;
        const long long u = uend - 1 - it;
        const int k0 = static_cast<int>(u % tiles_k) * kUnitK;
        tma_2d_g2s(xs + s * C::kXBytes, &tmap_x, k0, 0, full(s));
        tma_2d_g2s(xs + s * C::kXBytes + BM * 128, &tmap_x, k0 + 64, 0, full(s));
      };
      const int pre = nunits < S ? nunits : S;
      for (int it = 0; it < pre; ++it) issue_ws(it);
      if (!p.use_ticket) pdl_wait();  // X and the workspace belong to the previous kernel
      for (int it = 0; it < pre; ++it) issue_x(it);
      for (int it = pre; it < nunits; ++it) {
        const int s = it % S;
        mbar_wait(empty(s), ((it / S) & 1) ^ 1);
        issue_ws(it);
        issue_x(it);
      }
    }
  } else {
    // ===================== consumers =====================
    fill_lut<BITS>(lut, p.vlut, threadIdx.x, kConsumerWarps * 32);
    if (!p.use_ticket) pdl_wait();
    named_bar_sync(1, kConsumerWarps * 32);

    const uint32_t lane4 = static_cast<uint32_t>(lane) * 4u;
    // ldmatrix source offset for this lane (X box rows = m, 128B-swizzled).
    uint32_t xoff[MT > 1 ? MT / 2 : 1];
    {
      const int box = warp >> 2;
      const int c0 = (warp & 3) * 2;
      if (MT == 1) {
        const int r = lane & 7;
        const int c = c0 + ((lane >> 3) & 1);
        xoff[0] = box * (BM * 128) + r * 128 + ((c ^ r) << 4);
      } else {
#pragma unroll
        for (int q = 0; q < (MT > 1 ? MT / 2 : 1); ++q) {
          const int mat = lane >> 3;
          const int r = q * 16 + (mat >> 1) * 8 + (lane & 7);
          const int c = c0 + (mat & 1);
          xoff[q] = box * (BM * 128) + r * 128 + ((c ^ (r & 7)) << 4);
        }
      }
    }

    float acc[MT][4][4];
    for (int it = 0; it < nunits; ++it) {
      const long long u = uend - 1 - it;
      const long long tile = u / tiles_k;
      const int kt = static_cast<int>(u % tiles_k);
      if (it == 0 || kt == tiles_k - 1) {
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
          for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int r = 0; r < 4; ++r) acc[mt][j][r] = 0.f;
      }
      const int s = it % S;
      mbar_wait(full(s), (it / S) & 1);

      // ---- stage -> registers ----
      const uint32_t wst = ws + s * C::kUnitBytes;
      const int slot = warp * 32 + lane;
      LaneBits<BITS> lb;
      if constexpr (BITS == 4) {
        lb.w = lds128(wst + slot * 16);
      } else if constexpr (BITS == 2) {
        lb.w = lds64(wst + slot * 8);
      } else {
        lb.hi = lds64(wst + slot * 8);
        lb.lo = lds32(wst + 2048 + slot * 4);
      }
      const int gl = (kt * kUnitK + 16 * warp) / group - (kt * kUnitK) / group;
      const uint4 sq = lds128(ss + s * C::kScBytes + gl * 128 + (lane >> 2) * 16);
      uint32_t bf[MT][2];
      const uint32_t xst = xs + s * C::kXBytes;
      if constexpr (MT == 1) {
        ldsm_x2(xst + xoff[0], bf[0][0], bf[0][1]);
      } else {
#pragma unroll
        for (int q = 0; q < MT / 2; ++q)
          ldsm_x4(xst + xoff[q], bf[2 * q][0], bf[2 * q][1], bf[2 * q + 1][0], bf[2 * q + 1][1]);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(empty(s));

      // ---- dequant + MMA ----
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t sw = j == 0 ? sq.x : j == 1 ? sq.y : j == 2 ? sq.z : sq.w;
        uint32_t a[4];
        lut_dequant4(atom_index_bytes<BITS>(lb, j), lane4, lut, dup_lo(sw), dup_hi(sw), a);
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) mma_16816(acc[mt][j], a, bf[mt][0], bf[mt][1]);
      }

      if (it != nunits - 1 && kt != 0) continue;

      // ---- segment end: deterministic CTA reduction (tree over warps) ----
      float* accf = &acc[0][0][0];
      auto red_addr = [&](int sl, int i) {
        return red + ((sl * C::kFrag + i) * 32 + lane) * 4u;
      };
#pragma unroll
      for (int half = 4; half >= 1; half >>= 1) {
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

      if (warp == 0) {
        const long long t0 = tile * tiles_k;
        const bool started = ubeg <= t0;
        const bool finished = uend >= t0 + tiles_k;
        float* my_slot = p.slots + static_cast<size_t>(wid) * C::kFrag * 32;
        if (!finished) {
          // contributor: publish the fp32 partial, then release-add the
          // finisher's flag.
#pragma unroll
          for (int i = 0; i < C::kFrag; ++i) my_slot[i * 32 + lane] = accf[i];
          __threadfence();
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
            // ((c_first + c_next) + ...) + own, element by element
#pragma unroll
            for (int i = 0; i < C::kFrag; ++i) {
              float sum = 0.f;
              bool have = false;
              for (int c = first; c < wid; ++c) {
                if (range_lo(c + 1, U, P) <= range_lo(c, U, P)) continue;
                const float v = __ldcg(p.slots + (static_cast<size_t>(c) * C::kFrag + i) * 32 + lane);
                sum = have ? sum + v : v;
                have = true;
              }
              accf[i] = sum + accf[i];
            }
            __syncwarp();
            if (lane == 0) *reinterpret_cast<volatile uint32_t*>(p.flags + wid) = 0u;
          }
          // write Y (f16, RNE)
          const int g = lane >> 2, t = lane & 3;
          const long long ncol0 = tile * kUnitN;
#pragma unroll
          for (int mt = 0; mt < MT; ++mt)
#pragma unroll
            for (int j = 0; j < 4; ++j)
#pragma unroll
              for (int r = 0; r < 4; ++r) {
                const int row = mt * 8 + 2 * t + (r & 1);
                const long long col = ncol0 + 16 * j + g + 8 * (r >> 1);
                if (row < p.m && col < p.n)
                  p.y[static_cast<size_t>(row) * p.n + col] = __float2half_rn(acc[mt][j][r]);
              }
        }
      }
    }
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

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------

namespace {

[[noreturn]] void cuda_fail(const char* what, cudaError_t e) {
  throw flutesim::CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}
#define FLUTE_CUDA(call)                      \
  do {                                        \
    cudaError_t e_ = (call);                  \
    if (e_ != cudaSuccess) cuda_fail(#call, e_); \
  } while (0)

using EncodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                 const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                 const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                 CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiled encode_fn() {
  static EncodeTiled fn = [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q{};
    const cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q);
    if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || ptr == nullptr) {
      throw flutesim::CudaError("cuTensorMapEncodeTiled entry point unavailable");
    }
    return reinterpret_cast<EncodeTiled>(ptr);
  }();
  return fn;
}

CUtensorMap make_x_map(const void* x, int m, int k, int box_rows) {
  CUtensorMap map;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(k), static_cast<cuuint64_t>(m)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(k) * 2};
  const cuuint32_t box[2] = {64u, static_cast<cuuint32_t>(box_rows)};
  const cuuint32_t estr[2] = {1u, 1u};
  const CUresult r = encode_fn()(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void*>(x),
                                 dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                 CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    throw flutesim::InputError("X tensor map rejected (x must be 16-byte aligned, k % 8 == 0), code " +
                               std::to_string(static_cast<int>(r)));
  }
  return map;
}

struct DevProps {
  int sms = 0;
  size_t smem_optin = 0;
  int major = 0;
};

const DevProps& props() {
  static thread_local int cached_dev = -1;
  static thread_local DevProps pr;
  int dev = 0;
  FLUTE_CUDA(cudaGetDevice(&dev));
  if (dev != cached_dev) {
    cudaDeviceProp dp{};
    FLUTE_CUDA(cudaGetDeviceProperties(&dp, dev));
    if (dp.major != 10) {
      throw flutesim::CudaError("flute-b200 kernels need an sm_100 (Blackwell) device; found sm_" +
                                std::to_string(dp.major) + std::to_string(dp.minor));
    }
    pr.sms = dp.multiProcessorCount;
    pr.smem_optin = dp.sharedMemPerBlockOptin;
    pr.major = dp.major;
    cached_dev = dev;
  }
  return pr;
}

int bm_for(int m) { return m <= 8 ? 8 : m <= 16 ? 16 : 32; }

template <int BITS, int BM>
int stages_for() {
  const size_t cap = props().smem_optin;
  int s = kMaxStages;
  while (s > 2 && Cfg<BITS, BM>::smem_bytes(s) > cap) --s;
  return s;
}

template <int BITS, int BM>
void launch_impl(const GemmArgs& a, int m_rows, const void* x, void* y, int workers,
                 long long units, int tiles_k, int gp) {
  using Cf = Cfg<BITS, BM>;
  static thread_local int configured_dev = -1;
  int dev = 0;
  FLUTE_CUDA(cudaGetDevice(&dev));
  const int S = stages_for<BITS, BM>();
  const size_t smem = Cf::smem_bytes(S);
  if (configured_dev != dev) {
    FLUTE_CUDA(cudaFuncSetAttribute(qgemm_mma_kernel<BITS, BM>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(smem)));
    configured_dev = dev;
  }
  const CUtensorMap map = make_x_map(x, m_rows, a.k, BM);
  KParams kp{};
  kp.w = static_cast<const uint8_t*>(a.w);
  kp.sc = static_cast<const uint8_t*>(a.scales);
  kp.vlut = static_cast<const uint32_t*>(a.vlut);
  kp.y = static_cast<__half*>(y);
  const size_t flag_bytes = (static_cast<size_t>(workers) + 2) * 4;
  const size_t flag_span = (flag_bytes + 255) / 256 * 256;
  kp.flags = static_cast<uint32_t*>(a.workspace);
  kp.slots = reinterpret_cast<float*>(static_cast<uint8_t*>(a.workspace) + flag_span);
  kp.m = m_rows;
  kp.n = a.n;
  kp.tiles_k = tiles_k;
  kp.group = a.group;
  kp.gp = gp;
  kp.units = units;
  kp.workers = workers;
  kp.stages = S;
  kp.use_ticket = workers > props().sms ? 1 : 0;

  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(workers));
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = static_cast<cudaStream_t>(a.stream);
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  FLUTE_CUDA(cudaLaunchKernelEx(&cfg, qgemm_mma_kernel<BITS, BM>, map, kp));
}

template <int BITS>
void launch_bits(const GemmArgs& a, int m_rows, const void* x, void* y, int workers,
                 long long units, int tiles_k, int gp) {
  switch (bm_for(m_rows)) {
    case 8: launch_impl<BITS, 8>(a, m_rows, x, y, workers, units, tiles_k, gp); break;
    case 16: launch_impl<BITS, 16>(a, m_rows, x, y, workers, units, tiles_k, gp); break;
    default: launch_impl<BITS, 32>(a, m_rows, x, y, workers, units, tiles_k, gp); break;
  }
}

}  // namespace

int device_count() {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
  return n;
}

int sm_count(int device) {
  int v = 0;
  FLUTE_CUDA(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device));
  return v;
}

int max_workers(int m) {
  (void)m;
  return props().sms;  // one CTA per SM (smem-bound occupancy of 1)
}

int default_workers(int m, int k, int n, int bits) {
  (void)m;
  (void)bits;
  const long long units =
      static_cast<long long>((k + kUnitK - 1) / kUnitK) * ((n + kUnitN - 1) / kUnitN);
  return static_cast<int>(std::min<long long>(units, props().sms));
}

size_t workspace_bytes(int m, int workers) {
  const int bm = bm_for(std::min(m, 32));
  const size_t flag_bytes = (static_cast<size_t>(workers) + 2) * 4;
  const size_t flag_span = (flag_bytes + 255) / 256 * 256;
  return flag_span + static_cast<size_t>(workers) * (bm / 8) * 16 * 32 * 4;
}

void qgemm(const GemmArgs& a) {
  if (a.m < 1) throw flutesim::ConfigError("qgemm: m must be >= 1");
  if (a.bits < 2 || a.bits > 4) throw flutesim::ConfigError("qgemm: bits must be 2, 3 or 4");
  if (a.k % 16 != 0 || a.n % 16 != 0 || a.k < 16 || a.n < 16)
    throw flutesim::ConfigError("qgemm: k and n must be positive multiples of 16");
  if (!a.x || !a.w || !a.scales || !a.vlut || !a.y || !a.workspace)
    throw flutesim::InputError("qgemm: null device pointer");
  const int kp = (a.k + kUnitK - 1) / kUnitK * kUnitK;
  const int np = (a.n + kUnitN - 1) / kUnitN * kUnitN;
  if (kp % a.group != 0) throw flutesim::ConfigError("qgemm: padded k not divisible by group");
  const int tiles_k = kp / kUnitK;
  const long long units = static_cast<long long>(tiles_k) * (np / kUnitN);
  int workers = a.workers > 0 ? a.workers : default_workers(a.m, a.k, a.n, a.bits);
  if (a.workspace_bytes < workspace_bytes(a.m, workers))
    throw flutesim::InputError("qgemm: workspace too small");
  const int gp = kp / a.group;
  // M > 32: 32-row chunks, stream-ordered on one workspace.
  for (int r0 = 0; r0 < a.m; r0 += 32) {
    const int rows = std::min(32, a.m - r0);
    const void* x = static_cast<const uint8_t*>(a.x) + static_cast<size_t>(r0) * a.k * 2;
    void* y = static_cast<uint8_t*>(a.y) + static_cast<size_t>(r0) * a.n * 2;
    switch (a.bits) {
      case 2: launch_bits<2>(a, rows, x, y, workers, units, tiles_k, gp); break;
      case 3: launch_bits<3>(a, rows, x, y, workers, units, tiles_k, gp); break;
      default: launch_bits<4>(a, rows, x, y, workers, units, tiles_k, gp); break;
    }
  }
}

// ---------------------------------------------------------------------------
// Device self-check: run the GEMM's own dequant routine over every pair.
// ---------------------------------------------------------------------------

template <int BITS>
__global__ void dequant_all_kernel(const uint32_t* __restrict__ vlut, const uint16_t* __restrict__ scales,
                                   int n_scales, uint32_t* __restrict__ out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  constexpr int NP = 1 << (2 * BITS);
  const uint32_t lut = smem_u32(smem);
  fill_lut<BITS>(lut, vlut, threadIdx.x, blockDim.x);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  // Each (scale, group of 16*32 device indices) is one warp task.
  const int per_task = 16 * 32;
  const int tasks_per_scale = (NP + per_task - 1) / per_task;
  for (int task = gw; task < n_scales * tasks_per_scale; task += nw) {
    const int si = task / tasks_per_scale;
    const int d0 = (task % tasks_per_scale) * per_task + lane * 16;
    uint32_t d[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) d[q] = static_cast<uint32_t>((d0 + q) % NP);
    LaneBits<BITS> lb;
    if constexpr (BITS == 4) {
      uint32_t wv[4];
#pragma unroll
      for (int j = 0; j < 4; ++j)
        wv[j] = d[4 * j] | (d[4 * j + 1] << 8) | (d[4 * j + 2] << 16) | (d[4 * j + 3] << 24);
      lb.w = make_uint4(wv[0], wv[1], wv[2], wv[3]);
    } else {
      uint32_t hw[2] = {0u, 0u}, lo = 0u;
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int pp = 0; pp < 4; ++pp) {
          const uint32_t e = d[4 * j + pp];
          const uint32_t nib = BITS == 2 ? e : (e >> 2);
          hw[j >> 1] |= nib << (8 * pp + 4 * (j & 1));
          if (BITS == 3) lo |= (e & 3u) << (8 * pp + 2 * j);
        }
      if constexpr (BITS == 2) {
        lb.w = make_uint2(hw[0], hw[1]);
      } else {
        lb.hi = make_uint2(hw[0], hw[1]);
        lb.lo = lo;
      }
    }
    const uint32_t s = scales[si];
    const uint32_t sw = s | (s << 16);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      uint32_t a[4];
      lut_dequant4(atom_index_bytes<BITS>(lb, j), static_cast<uint32_t>(lane) * 4u, lut, dup_lo(sw),
                   dup_hi(sw), a);
#pragma unroll
      for (int pp = 0; pp < 4; ++pp) {
        const int q = 4 * j + pp;
        if (d0 + q < NP) {
          const uint32_t e = d[q];
          uint32_t ref = e;
          if (BITS == 3) {  // device index -> reference pair (ik << 3 | ik1)
            const uint32_t ik = (((e >> 4) & 3u) << 1) | ((e >> 1) & 1u);
            const uint32_t ik1 = (((e >> 2) & 3u) << 1) | (e & 1u);
            ref = (ik << 3) | ik1;
          }
          out[static_cast<size_t>(si) * NP + ref] = a[pp];
        }
      }
    }
  }
}

struct DevBuf {
  void* p = nullptr;
  explicit DevBuf(size_t n) { FLUTE_CUDA(cudaMalloc(&p, n ? n : 1)); }
  ~DevBuf() { cudaFree(p); }
};

void dequant_all(const uint32_t* vlut_words, int bits, const uint16_t* scales, int n_scales,
                 uint32_t* out_host) {
  if (bits < 2 || bits > 4) throw flutesim::ConfigError("dequant_all: bits must be 2..4");
  if (n_scales < 1) throw flutesim::InputError("dequant_all: need at least one scale");
  (void)props();
  const int np = 1 << (2 * bits);
  DevBuf dv(np * 4), ds(n_scales * 2), dout(static_cast<size_t>(n_scales) * np * 4);
  FLUTE_CUDA(cudaMemcpy(dv.p, vlut_words, np * 4, cudaMemcpyHostToDevice));
  FLUTE_CUDA(cudaMemcpy(ds.p, scales, n_scales * 2, cudaMemcpyHostToDevice));
  const int lut_bytes = np * kLutRowBytes;
  const int blocks = std::min(1024, n_scales);
  auto run = [&](auto kern) {
    FLUTE_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, lut_bytes));
    kern<<<blocks, 256, lut_bytes>>>(static_cast<const uint32_t*>(dv.p),
                                     static_cast<const uint16_t*>(ds.p), n_scales,
                                     static_cast<uint32_t*>(dout.p));
  };
  if (bits == 2) run(dequant_all_kernel<2>);
  else if (bits == 3) run(dequant_all_kernel<3>);
  else run(dequant_all_kernel<4>);
  FLUTE_CUDA(cudaGetLastError());
  FLUTE_CUDA(cudaMemcpy(out_host, dout.p, static_cast<size_t>(n_scales) * np * 4,
                        cudaMemcpyDeviceToHost));
}

// ---------------------------------------------------------------------------
// mma_fragment on the tensor cores (reference mma.cpp:10-30 simulates this).
// ---------------------------------------------------------------------------

__global__ void mma_fragment_kernel(const __half* __restrict__ A, const __half* __restrict__ B,
                                    float* __restrict__ Cm, int m, int n, int k) {
  const int lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  auto a_at = [&](int r, int c) -> uint32_t {
    return (r < m && c < k) ? __half_as_ushort(A[r * k + c]) : 0u;
  };
  auto b_at = [&](int r, int c) -> uint32_t {
    return (r < k && c < n) ? __half_as_ushort(B[r * n + c]) : 0u;
  };
  for (int m0 = 0; m0 < m; m0 += 16)
    for (int n0 = 0; n0 < n; n0 += 8) {
      float d[4];
      const int rr[4] = {g, g, g + 8, g + 8};
      const int cc[4] = {2 * t, 2 * t + 1, 2 * t, 2 * t + 1};
      for (int r = 0; r < 4; ++r) {
        const int row = m0 + rr[r], col = n0 + cc[r];
        d[r] = (row < m && col < n) ? Cm[row * n + col] : 0.f;
      }
      for (int k0 = 0; k0 < k; k0 += 16) {
        uint32_t a[4];
        a[0] = a_at(m0 + g, k0 + 2 * t) | (a_at(m0 + g, k0 + 2 * t + 1) << 16);
        a[1] = a_at(m0 + g + 8, k0 + 2 * t) | (a_at(m0 + g + 8, k0 + 2 * t + 1) << 16);
        a[2] = a_at(m0 + g, k0 + 2 * t + 8) | (a_at(m0 + g, k0 + 2 * t + 9) << 16);
        a[3] = a_at(m0 + g + 8, k0 + 2 * t + 8) | (a_at(m0 + g + 8, k0 + 2 * t + 9) << 16);
        const uint32_t b0 = b_at(k0 + 2 * t, n0 + g) | (b_at(k0 + 2 * t + 1, n0 + g) << 16);
        const uint32_t b1 = b_at(k0 + 2 * t + 8, n0 + g) | (b_at(k0 + 2 * t + 9, n0 + g) << 16);
        mma_16816(d, a, b0, b1);
      }
      for (int r = 0; r < 4; ++r) {
        const int row = m0 + rr[r], col = n0 + cc[r];
        if (row < m && col < n) Cm[row * n + col] = d[r];
      }
    }
}

void mma_fragment(const uint16_t* a, const uint16_t* b, float* c, int m, int n, int k) {
  (void)props();
  DevBuf da(static_cast<size_t>(m) * k * 2), db(static_cast<size_t>(k) * n * 2),
      dc(static_cast<size_t>(m) * n * 4);
  FLUTE_CUDA(cudaMemcpy(da.p, a, static_cast<size_t>(m) * k * 2, cudaMemcpyHostToDevice));
  FLUTE_CUDA(cudaMemcpy(db.p, b, static_cast<size_t>(k) * n * 2, cudaMemcpyHostToDevice));
  FLUTE_CUDA(cudaMemcpy(dc.p, c, static_cast<size_t>(m) * n * 4, cudaMemcpyHostToDevice));
  mma_fragment_kernel<<<1, 32>>>(static_cast<const __half*>(da.p), static_cast<const __half*>(db.p),
                                 static_cast<float*>(dc.p), m, n, k);
  FLUTE_CUDA(cudaGetLastError());
  FLUTE_CUDA(cudaMemcpy(c, dc.p, static_cast<size_t>(m) * n * 4, cudaMemcpyDeviceToHost));
}

// ---------------------------------------------------------------------------
// buffers
// ---------------------------------------------------------------------------

void* dev_alloc(size_t bytes) {
  void* p = nullptr;
  FLUTE_CUDA(cudaMalloc(&p, bytes ? bytes : 1));
  return p;
}
void dev_free(void* p) {
  if (p) cudaFree(p);
}
void h2d(void* dst, const void* src, size_t bytes, void* stream) {
  FLUTE_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, static_cast<cudaStream_t>(stream)));
}
void d2h(void* dst, const void* src, size_t bytes, void* stream) {
  FLUTE_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, static_cast<cudaStream_t>(stream)));
}
void dev_zero(void* p, size_t bytes, void* stream) {
  FLUTE_CUDA(cudaMemsetAsync(p, 0, bytes, static_cast<cudaStream_t>(stream)));
}
void stream_sync(void* stream) { FLUTE_CUDA(cudaStreamSynchronize(static_cast<cudaStream_t>(stream))); }

}  // namespace flute_dev
