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
#include <cstdlib>
#include <string>
#include <type_traits>

#include "dequant.cuh"
#include "device_api.h"
#include "flutesim/errors.hpp"
#include "ptx.cuh"

namespace flute_dev {

namespace tc {

constexpr int kDqWarps = 8;
constexpr int kTmaWarp = 8;
constexpr int kMmaWarp = 9;
constexpr int kThreads = 320;
constexpr int kUnitK = 128;
constexpr int kMaxStages = 4;

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
  int stages;
  int ng;  // scale groups per unit in a stage's scale block (>= 1)
  uint32_t lut_bytes, bar_off, stage_off, stage_bytes;
};

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

__device__ __forceinline__ void umma_f16(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                         uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
      ::"r"(d_tmem), "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void umma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
               : "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void sts32(uint32_t addr, uint32_t v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, "
      "%12, %13, %14, %15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// KD = stage depth: 128 (one unit per stage, two 64-k swizzle atoms) or 64
// (half a unit: one atom, so a BN = 256 X tile still double-buffers within
// shared memory; the 8 dequant warps then split as 2 units x 4 k-steps).
template <int BITS, int BN, int KD>
__global__ void __launch_bounds__(kThreads, 1)
    qgemm_tc_kernel(const __grid_constant__ CUtensorMap tmap_x, const Params p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  static_assert(KD == 128 || KD == 64, "stage depth");
  constexpr int kAtoms = KD / 64;             // 64-k swizzle atoms per stage
  constexpr int kSubBytes = BITS * 1024;      // one unit's packed weights
  constexpr int kStageW = kSubBytes * KD / 128;  // per unit per stage
  constexpr uint32_t kABytes = kAtoms * 16384;   // kAtoms 64-k swizzle atoms of 128 rows
  constexpr uint32_t kXBox = BN * 128;      // one 64-k box of BN rows
  constexpr uint32_t kWOff = kABytes + kAtoms * kXBox;
  constexpr uint32_t kSOff = kWOff + 2 * kStageW;

  const uint32_t base = smem_u32(smem);
  const uint32_t lut = base;
  const uint32_t bars = base + p.bar_off;
  const int S = p.stages;
  auto full_w = [&](int s) { return bars + 8 * s; };
  auto full_x = [&](int s) { return bars + 8 * (kMaxStages + s); };
  auto a_ready = [&](int s) { return bars + 8 * (2 * kMaxStages + s); };
  auto empty = [&](int s) { return bars + 8 * (3 * kMaxStages + s); };
  const uint32_t acc_full = bars + 8 * (4 * kMaxStages);
  const uint32_t tmem_slot = acc_full + 8;  // tcgen05.alloc writes the TMEM base here
  auto stage = [&](int s) { return base + p.stage_off + s * p.stage_bytes; };

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int pair = blockIdx.x;  // 128-column tile = units' n-tiles 2*pair, 2*pair+1
  const int m0 = blockIdx.y * BN;
  const int z = blockIdx.z;
  const int kt_lo = z * p.tiles_k / p.splits;
  const int kt_hi = (z + 1) * p.tiles_k / p.splits;
  const int nk = (kt_hi - kt_lo) * (128 / KD);  // stages
  const int nt0 = 2 * pair;
  const bool has_u1 = nt0 + 1 < p.tiles_n;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(full_w(s), 1);
      mbar_init(full_x(s), 1);
      mbar_init(a_ready(s), kDqWarps);
      // the MMA commit (A / X read by the tensor core) + every dequant lane
      // (its reads of the stage's weights and scales done)
      mbar_init(empty(s), 1 + kDqWarps * 32);
    }
    mbar_init(acc_full, 1);
    fence_mbar_init();
  }
  if (warp == kMmaWarp) {
    // TMEM accumulator: BN fp32 columns x 128 lanes
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tmem_slot),
                 "n"(BN < 32 ? 32 : BN)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(smem + (tmem_slot - base));
  pdl_launch_dependents();

  if (warp == kTmaWarp) {
    // ===================== TMA producer =====================
    if (elect_one()) {
      prefetch_tmap(&tmap_x);
      const uint64_t pol = policy_evict_first();
      const int units_pair = has_u1 ? 2 : 1;
      for (int i = 0, s = 0, ph = 0; i < nk; ++i) {
        const int kt = kt_lo + i / (128 / KD);
        const int half = KD == 64 ? (i & 1) : 0;  // which 64-k half of the unit
        if (i >= S) mbar_wait(empty(s), ph ^ 1);
        const uint32_t st = stage(s);
        const int glo = (kt * kUnitK) >> p.group_shift;
        const uint32_t sb = p.ng * 128;
        mbar_arrive_expect_tx(full_w(s), units_pair * (kStageW + sb));
        for (int u = 0; u < units_pair; ++u) {
          const size_t unit = static_cast<size_t>(nt0 + u) * p.tiles_k + kt;
          const uint8_t* wu = p.w + unit * kSubBytes;
          if constexpr (KD == 128) {
            bulk_g2s_hint(st + kWOff + u * kStageW, wu, kSubBytes, full_w(s), pol);
          } else if constexpr (BITS == 3) {
            // k-steps 4h..4h+3: 2-bit plane bytes [1024h, +1024), 1-bit [2048 + 512h, +512)
            bulk_g2s_hint(st + kWOff + u * kStageW, wu + 1024 * half, 1024, full_w(s), pol);
            bulk_g2s_hint(st + kWOff + u * kStageW + 1024, wu + 2048 + 512 * half, 512, full_w(s), pol);
          } else {
            bulk_g2s_hint(st + kWOff + u * kStageW, wu + kStageW * half, kStageW, full_w(s), pol);
          }
          bulk_g2s(st + kSOff + u * sb, p.sc + (static_cast<size_t>(nt0 + u) * p.gp + glo) * 128, sb,
                   full_w(s));
        }
        if (i == 0) pdl_wait();  // X belongs to the previous kernel in the stream
        mbar_arrive_expect_tx(full_x(s), kAtoms * kXBox);
#pragma unroll
        for (int a = 0; a < kAtoms; ++a)
          tma_2d_g2s(st + kABytes + a * kXBox, &tmap_x, kt * kUnitK + 64 * (half + a), m0, full_x(s));
        if (++s == S) {
          s = 0;
          ph ^= 1;
        }
      }
    }
  } else if (warp == kMmaWarp) {
    // ===================== MMA issuer =====================
    constexpr uint32_t idesc = instr_desc<BN>();
    for (int i = 0, s = 0, ph = 0; i < nk; ++i) {
      mbar_wait(full_x(s), ph);
      mbar_wait(a_ready(s), ph);
      tc_fence_after();
      const uint32_t st = stage(s);
      if (elect_one()) {
#pragma unroll
        for (int a = 0; a < kAtoms; ++a)
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const uint64_t ad = smem_desc_sw128(st + a * 16384 + kk * 32);
            const uint64_t bd = smem_desc_sw128(st + kABytes + a * kXBox + kk * 32);
            umma_f16(tmem, ad, bd, idesc, (i | a | kk) != 0 ? 1u : 0u);
          }
        umma_commit(empty(s));  // smem stage free once these MMAs have read it
        if (i == nk - 1) umma_commit(acc_full);
      }
      __syncwarp();
      if (++s == S) {
        s = 0;
        ph ^= 1;
      }
    }
  } else {
    // ===================== dequant warps (0..7) =====================
    fill_lut<BITS, kDqWarps * 32>(lut, p.vlut, threadIdx.x);
    named_bar_sync(1, kDqWarps * 32);
    const uint32_t lane4 = static_cast<uint32_t>(lane) * 4u;
    // KD = 128: warp w owns k-step w of both units; KD = 64: k-step (w & 3) of
    // the stage's half of unit w >> 2 (local k-step kl within the stage)
    constexpr int kUnitsPerWarp = KD == 128 ? 2 : 1;
    const int kl = KD == 128 ? warp : (warp & 3);
    const int u0 = KD == 128 ? 0 : (warp >> 2);
    const int slot = kl * 32 + lane;  // this lane's slot within the stage's weight bytes
    const int g = lane >> 2, t = lane & 3;
    // A-tile byte offset of this lane's pair p of atom j, unit u (row n, k = kk, kk+1)
    auto a_off = [&](int u, int j, int pp) -> uint32_t {
      const int n = 64 * u + 16 * j + g + 8 * (pp & 1);
      const int kk = 16 * kl + 2 * t + 8 * (pp >> 1);
      const int at = kk >> 6, kin = kk & 63;
      return static_cast<uint32_t>(at * 16384 + (n >> 3) * 1024 + (n & 7) * 128 +
                                   ((((kin >> 3) ^ (n & 7))) << 4) + (kin & 7) * 2);
    };
    uint32_t aoff[kUnitsPerWarp][4][4];
#pragma unroll
    for (int uu = 0; uu < kUnitsPerWarp; ++uu)
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int pp = 0; pp < 4; ++pp) aoff[uu][j][pp] = a_off(u0 + uu, j, pp);
    const uint32_t s_lane = (lane >> 2) * 16;
    for (int i = 0, s = 0, ph = 0; i < nk; ++i) {
      const int kt = kt_lo + i / (128 / KD);
      const int kstep = KD == 128 ? kl : kl + 4 * (i & 1);  // k-step within the unit
      mbar_wait(full_w(s), ph);
      const uint32_t st = stage(s);
      const int gl = (((kt << 7) + 16 * kstep) >> p.group_shift) - ((kt << 7) >> p.group_shift);
#pragma unroll
      for (int uu = 0; uu < kUnitsPerWarp; ++uu) {
        const int u = u0 + uu;
        if (u == 1 && !has_u1) break;
        const uint32_t wr = st + kWOff + u * kStageW;
        LaneBits<BITS> lb;
        if constexpr (BITS == 4) {
          lb.w = lds128(wr + slot * 16);
        } else if constexpr (BITS == 2) {
          lb.w = lds64(wr + slot * 8);
        } else {
          lb.hi = lds64(wr + slot * 8);
          lb.lo = lds32(wr + kStageW * 2 / 3 + slot * 4);  // 1-bit plane after the 2-bit plane
        }
        const uint4 sq = lds128(st + kSOff + u * p.ng * 128 + gl * 128 + s_lane);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint32_t scw = j == 0 ? sq.x : j == 1 ? sq.y : j == 2 ? sq.z : sq.w;
          uint32_t a[4];
          lut_dequant4(atom_index_bytes<BITS>(lb, j), lane4, lut, scw, a);
#pragma unroll
          for (int pp = 0; pp < 4; ++pp) sts32(st + aoff[uu][j][pp], a[pp]);
        }
      }
      fence_proxy_async_smem();  // generic-proxy A stores -> visible to the tensor core
      __syncwarp();
      if (lane == 0) mbar_arrive(a_ready(s));
      mbar_arrive(empty(s));
      if (++s == S) {
        s = 0;
        ph ^= 1;
      }
    }
    // ===================== epilogue (warps 0..3) =====================
    if (warp < 4) {
      mbar_wait(acc_full, 0);
      tc_fence_after();
      const int n = pair * 128 + warp * 32 + lane;  // this thread's TMEM lane = output column
      const uint32_t trow = tmem + (static_cast<uint32_t>(warp * 32) << 16);
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 16) {
        uint32_t v[16];
        tmem_ld16(trow + c0, v);
        if (n < p.n) {
#pragma unroll
          for (int q = 0; q < 16; ++q) {
            const int m = m0 + c0 + q;
            if (m < p.m) {
              const float f = __uint_as_float(v[q]);
              if (p.splits > 1)
                p.part[(static_cast<size_t>(z) * p.m + m) * p.n + n] = f;
              else
                p.y[static_cast<size_t>(m) * p.n + n] = __float2half_rn(f);
            }
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarp) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "n"(BN < 32 ? 32 : BN)
                 : "memory");
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

template <int BITS, int BN, int KD>
void launch_tc(const GemmArgs& a, const TcPlan& pl, cudaStream_t stream) {
  static thread_local int configured = -1;
  int dev = 0;
  FLUTE_TC_CUDA(cudaGetDevice(&dev));
  auto kern = tc::qgemm_tc_kernel<BITS, BN, KD>;
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
  cfg.blockDim = dim3(tc::kThreads);
  cfg.dynamicSmemBytes = pl.smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  FLUTE_TC_CUDA(cudaLaunchKernelEx(&cfg, kern, map, pl.prm));
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

bool tc_enabled(int m) { return m >= 64 && std::getenv("FLUTE_NO_TC") == nullptr; }

void qgemm_tc(const GemmArgs& a, int tiles_k, int tiles_n, int gp, int sms, bool zero_part,
              void* part, size_t part_bytes) {
  TcPlan pl;
  pl.zero_part = zero_part;
  pl.bn = tc_bn(a.m, tiles_n, sms);
  if (pl.bn != 64 && pl.bn != 128 && pl.bn != 256) throw flutesim::ConfigError("FLUTE_TC_BN must be 64, 128 or 256");
  const int kd = pl.bn == 256 ? 64 : 128;
  const long tiles = static_cast<long>((tiles_n + 1) / 2) * ((a.m + pl.bn - 1) / pl.bn);
  pl.splits = static_cast<int>(
      std::max<long>(1, std::min<long>(std::min(tiles_k, 8), sms / std::max<long>(tiles, 1))));
  if (const char* f = std::getenv("FLUTE_TC_SPLITS")) pl.splits = std::max(1, std::min(tiles_k, std::atoi(f)));
  while (pl.splits > 1 && static_cast<size_t>(pl.splits) * a.m * a.n * 4 > part_bytes) --pl.splits;
  const int ng = std::max(1, 128 >> __builtin_ctz(static_cast<unsigned>(a.group)));
  const size_t lut = static_cast<size_t>(1u << (2 * a.bits)) * kLutRowBytes;
  const size_t bar_off = lut;
  const size_t stage_off = (bar_off + 8 * (4 * tc::kMaxStages + 2) + 1023) / 1024 * 1024;
  const size_t atoms = kd / 64;
  const size_t stage_bytes = ((atoms * 16384 + atoms * static_cast<size_t>(pl.bn) * 128 +
                               2 * static_cast<size_t>(a.bits) * 1024 * kd / 128 + 2 * ng * 128) +
                              1023) / 1024 * 1024;
  int optin = 0, dev = 0;
  FLUTE_TC_CUDA(cudaGetDevice(&dev));
  FLUTE_TC_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  pl.stages = static_cast<int>(std::min<size_t>(tc::kMaxStages, (optin - stage_off) / stage_bytes));
  if (pl.stages < 2) throw flutesim::InternalError("qgemm_tc: shared-memory plan has < 2 stages");
  pl.smem = stage_off + pl.stages * stage_bytes;
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
  p.stages = pl.stages;
  p.ng = ng;
  p.lut_bytes = static_cast<uint32_t>(lut);
  p.bar_off = static_cast<uint32_t>(bar_off);
  p.stage_off = static_cast<uint32_t>(stage_off);
  p.stage_bytes = static_cast<uint32_t>(stage_bytes);
  cudaStream_t st = static_cast<cudaStream_t>(a.stream);
  auto go = [&](auto bits_tag) {
    constexpr int B = decltype(bits_tag)::value;
    if (pl.bn == 256) launch_tc<B, 256, 64>(a, pl, st);
    else if (pl.bn == 128) launch_tc<B, 128, 128>(a, pl, st);
    else launch_tc<B, 64, 128>(a, pl, st);
  };
  switch (a.bits) {
    case 2: go(std::integral_constant<int, 2>{}); break;
    case 3: go(std::integral_constant<int, 3>{}); break;
    default: go(std::integral_constant<int, 4>{}); break;
  }
}

}  // namespace flute_dev
