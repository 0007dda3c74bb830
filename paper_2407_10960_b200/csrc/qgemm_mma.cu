// flute-b200 — host launcher of the memory-bound LUT-GEMM (kernel in
// qgemm_kernel.cuh) plus the device self-check kernels (exhaustive dequant,
// tensor-core mma_fragment) and small CUDA runtime helpers.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <string>

#include "dequant.cuh"
#include "device_api.h"
#include "flutesim/errors.hpp"
#include "ptx.cuh"
#include "qgemm_kernel.cuh"

namespace flute_dev {

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

// X [m][k] f16.  k % 64 == 0: a 3-D view {64 k, m, k/64 chunks} so one TMA op
// brings a unit's two 64-wide chunks; otherwise the plain 2-D view (two ops,
// zero fill past k).
CUtensorMap make_x_map(const void* x, int m, int k, int box_rows, int box_chunks, bool three_d) {
  CUtensorMap map;
  const cuuint32_t estr[3] = {1u, 1u, 1u};
  CUresult r;
  if (three_d) {
    const cuuint64_t dims[3] = {64u, static_cast<cuuint64_t>(m), static_cast<cuuint64_t>(k / 64)};
    const cuuint64_t strides[2] = {static_cast<cuuint64_t>(k) * 2, 128u};
    const cuuint32_t box[3] = {64u, static_cast<cuuint32_t>(box_rows),
                               static_cast<cuuint32_t>(box_chunks)};
    r = encode_fn()(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, const_cast<void*>(x), dims, strides,
                    box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else {
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(k), static_cast<cuuint64_t>(m)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(k) * 2};
    const cuuint32_t box[2] = {64u, static_cast<cuuint32_t>(box_rows)};
    r = encode_fn()(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void*>(x), dims, strides,
                    box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
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

// FLUTE_DEBUG_TIMES=1 (diag build): per-CTA %globaltimer stamps {start,
// producer issued, LUT ready, first stage ready, segment end, last segment
// end, exit, finisher acquired} followed by a per-stage trace of consumer
// warp 0: 64 stages x {wait begin, data ready, compute done}.
constexpr size_t kDbgPerCta = 16 + 64 * 3;
unsigned long long* g_dbg = nullptr;
int g_dbg_cap = 0;       // CTAs per slot
int g_dbg_slots = 1;     // FLUTE_DEBUG_TIMES=N: ring of N launches (no per-launch memset,
int g_dbg_next = 0;      // so programmatic-dependent launches still overlap)
unsigned long long* debug_times_buffer(int workers) {
  static const char* env = std::getenv("FLUTE_DEBUG_TIMES");
  if (!env) return nullptr;
  const int slots = std::max(1, std::atoi(env));
  const size_t slot_words = static_cast<size_t>(workers) * kDbgPerCta;
  if (g_dbg_cap < workers || g_dbg_slots != slots) {
    if (g_dbg) cudaFree(g_dbg);
    FLUTE_CUDA(cudaMalloc(&g_dbg, slot_words * slots * 8));
    FLUTE_CUDA(cudaMemset(g_dbg, 0, slot_words * slots * 8));
    g_dbg_cap = workers;
    g_dbg_slots = slots;
    g_dbg_next = 0;
  }
  if (slots == 1) FLUTE_CUDA(cudaMemset(g_dbg, 0, slot_words * 8));
  unsigned long long* b = g_dbg + static_cast<size_t>(g_dbg_next) * g_dbg_cap * kDbgPerCta;
  g_dbg_next = (g_dbg_next + 1) % slots;
  return b;
}

int bm_for(int m) { return m <= 8 ? 8 : m <= 16 ? 16 : 32; }

size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

// Shared memory available to one CTA when `occ` CTAs must fit on an SM.
size_t smem_cap(int occ) {
  static thread_local int dev_cached = -1;
  static thread_local size_t per_sm = 0, reserved = 0, optin = 0;
  int dev = 0;
  FLUTE_CUDA(cudaGetDevice(&dev));
  if (dev != dev_cached) {
    int v = 0;
    FLUTE_CUDA(cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev));
    per_sm = static_cast<size_t>(v);
    FLUTE_CUDA(cudaDeviceGetAttribute(&v, cudaDevAttrReservedSharedMemoryPerBlock, dev));
    reserved = static_cast<size_t>(v);
    optin = props().smem_optin;
    dev_cached = dev;
  }
  return std::min(optin, per_sm / static_cast<size_t>(occ) - reserved);
}

struct SmemPlan {
  uint32_t part_off = 0, part_stride = 0, stage_off = 0, stage_bytes = 0, x_bytes = 0, bar_off = 0;
  uint32_t recv_off = 0;
  int stages = 0;
  size_t total = 0;
};

// [vLUT (+ partial rows in its row gaps) | partials | barriers | stages...],
// stage = [X (1024-aligned, zero row last) | weights | scales].
template <int BITS, int BM, int UPS, int CW>
SmemPlan plan_smem(int m, int group, int cluster, size_t cap) {
  using Cf = Cfg<BITS, BM, UPS, CW>;
  SmemPlan pl;
  size_t off = Cf::kLutBytes;
  pl.part_off = static_cast<uint32_t>(off);
  pl.part_stride = 128;
  off += Cf::kPartBytes;
  pl.recv_off = static_cast<uint32_t>(off);  // cluster split-K receive buffer
  if (cluster > 1) off += static_cast<size_t>(cluster - 1) * Cf::kFrag * 128;
  pl.bar_off = static_cast<uint32_t>(off);
  off = align_up(off + Cf::kBarBytes, 1024);
  pl.stage_off = static_cast<uint32_t>(off);
  pl.x_bytes = static_cast<uint32_t>(align_up(2 * UPS * m * 128 + (m < BM ? 128 : 0), 1024));
  const int ng = UPS * std::max(1, kUnitK / group);
  pl.stage_bytes =
      static_cast<uint32_t>(align_up(pl.x_bytes + Cf::kWBytes + static_cast<size_t>(ng) * 128, 1024));
  const long fit = cap > off ? static_cast<long>((cap - off) / pl.stage_bytes) : 0;
  pl.stages = static_cast<int>(std::min<long>(kMaxStages, fit));
  pl.total = off + static_cast<size_t>(pl.stages) * pl.stage_bytes;
  return pl;
}

template <int BITS, int BM, int UPS, int OCC, int CW>
void launch_impl(const GemmArgs& a, int m_rows, const void* x, void* y, int workers,
                 long long units, int tiles_k, int gp, int cluster) {
  using Cf = Cfg<BITS, BM, UPS, CW>;
  static thread_local int configured_dev = -1;
  int dev = 0;
  FLUTE_CUDA(cudaGetDevice(&dev));
  const SmemPlan pl = plan_smem<BITS, BM, UPS, CW>(m_rows, a.group, cluster, smem_cap(OCC));
  if (pl.stages < 2) throw flutesim::InternalError("qgemm: shared-memory plan has < 2 stages");
  auto kern = qgemm_mma_kernel<BITS, BM, UPS, OCC, CW>;
  if (configured_dev != dev) {
    FLUTE_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(smem_cap(OCC))));
    configured_dev = dev;
  }
  const bool x3d = a.k % 64 == 0 && std::getenv("FLUTE_X2D") == nullptr;
  const CUtensorMap map = make_x_map(x, m_rows, a.k, m_rows, 2 * UPS, x3d);
  KParams kp{};
  kp.w = static_cast<const uint8_t*>(a.w);
  kp.sc = static_cast<const uint8_t*>(a.scales);
  kp.vlut = static_cast<const uint32_t*>(a.vlut);
  if (a.n_peers > 0) {
    // y points at the row-0 slot of this launch's row chunk in peer 0's buffer;
    // the same row offset applies to every peer
    const size_t row_off = static_cast<const uint8_t*>(y) - static_cast<const uint8_t*>(a.y_peers[0]);
    for (int i = 0; i < a.n_peers; ++i)
      kp.y_out[i] = reinterpret_cast<__half*>(static_cast<uint8_t*>(a.y_peers[i]) + row_off);
    kp.n_out = a.n_peers;
    kp.ldy = a.ldy;
    kp.ycol0 = a.ycol0;
  } else {
    kp.y_out[0] = static_cast<__half*>(y);
    kp.n_out = 1;
    kp.ldy = a.n;
    kp.ycol0 = 0;
  }
  const size_t flag_bytes = (static_cast<size_t>(workers) + 2) * 4;
  const size_t flag_span = (flag_bytes + 255) / 256 * 256;
  kp.flags = static_cast<uint32_t*>(a.workspace);
  kp.slots = reinterpret_cast<float*>(static_cast<uint8_t*>(a.workspace) + flag_span);
  kp.m = m_rows;
  kp.n = a.n;
  kp.tiles_k = tiles_k;
  kp.group_shift = __builtin_ctz(static_cast<unsigned>(a.group));
  kp.gp = gp;
  kp.units = static_cast<int>(units);
  kp.workers = workers;
  kp.stages = pl.stages;
  kp.use_ticket = cluster <= 1 && workers > props().sms * OCC ? 1 : 0;
  kp.cluster = cluster;
  kp.recv_off = pl.recv_off;
  kp.x3d = x3d ? 1 : 0;
  kp.part_off = pl.part_off;
  kp.part_stride = pl.part_stride;
  kp.stage_off = pl.stage_off;
  kp.stage_bytes = pl.stage_bytes;
  kp.x_bytes = pl.x_bytes;
  kp.bar_off = pl.bar_off;
  {
    static const char* d = std::getenv("FLUTE_DIAG");
    kp.diag = d ? std::atoi(d) : 0;
  }
  kp.dbg = debug_times_buffer(workers);
  (void)Cf::kWBytes;

  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(workers));
  cfg.blockDim = dim3(threads_for(CW));
  cfg.dynamicSmemBytes = pl.total;
  cfg.stream = static_cast<cudaStream_t>(a.stream);
  cudaLaunchAttribute attr[2];
  int na = 0;
  static const bool no_pdl = std::getenv("FLUTE_NO_PDL") != nullptr;
  if (!no_pdl) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  if (cluster > 1) {
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = static_cast<unsigned>(cluster);
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  FLUTE_CUDA(cudaLaunchKernelEx(&cfg, kern, map, kp));
}

// Per row-block: (stage depth UPS units, CTAs per SM the kernel is built for).
//   m <= 8 : UPS 2, OCC 2  (co-resident with the next launch)
//   m <= 16: UPS 1, OCC 2
//   m <= 32: UPS 2, OCC 1  (64 accumulator floats / lane: one CTA per SM)
// (A single 16-consumer-warp CTA per SM — CW = 16, OCC = 1 — was measured
// 10-30 % slower than two 8-warp CTAs on every configs[1] case.)
// Launch the <BITS, BM, UPS, OCC, CW> instantiation if its shared-memory plan
// keeps at least `min_stages` pipeline stages.
template <int BITS, int BM, int UPS, int OCC, int CW>
bool try_launch(int min_stages, const GemmArgs& a, int m_rows, const void* x, void* y,
                int workers, long long units, int tiles_k, int gp, int cluster) {
  if (plan_smem<BITS, BM, UPS, CW>(m_rows, a.group, cluster, smem_cap(OCC)).stages < min_stages)
    return false;
  launch_impl<BITS, BM, UPS, OCC, CW>(a, m_rows, x, y, workers, units, tiles_k, gp, cluster);
  return true;
}

template <int BITS>
void launch_bits(const GemmArgs& a, int m_rows, const void* x, void* y, int workers,
                 long long units, int tiles_k, int gp, int cluster) {
  // Measured on B200 (profiles/r1/README.md):
  //  * 4 consumer warps per CTA beat 8 (same CTA count): 5-11 % faster at
  //    M <= 16 — less shared-memory / issue contention per SM and half the
  //    partial sums to reduce per segment;
  //  * larger stages when >= 3 of them fit: W3 four units per stage for
  //    M <= 16 (two for 17..32), W2 four for M <= 8 and two for 9..16 (3-8 %
  //    faster); W4's 64 KB vLUT leaves room for two / one;
  //  * M = 17..32, W2/W3: two CTAs per SM (two 4-warp CTAs fit the register
  //    file; a launch hands its SM slots to the next one CTA at a time under
  //    PDL) — 7-11 % faster than one 8-warp CTA; W4 keeps one 8-warp CTA.
#define FLUTE_TRY(BM, UPS, OCC, CW, MIN) \
  if (try_launch<BITS, BM, UPS, OCC, CW>(MIN, a, m_rows, x, y, workers, units, tiles_k, gp, cluster)) return
  switch (bm_for(m_rows)) {
    case 8:
      // W3: four-unit stages, three of them if they fit, else two (the
      // 256-row table leaves room for only two at M > 1 or with a cluster
      // receive buffer; two four-unit stages measured 1-4 % faster than
      // three-plus two-unit ones: 14336x4096 M=1 10.72 -> 10.30 us)
      if constexpr (BITS == 3) {
        FLUTE_TRY(8, 4, 2, 4, 3);
        FLUTE_TRY(8, 4, 2, 4, 2);
      }
      // W4: four-unit stages, two of them (C1 4096^2 M=1 5.61 -> 5.51 us, 70B
      // layer 28.3 -> 27.3 us; W2 measured neutral)
      if constexpr (BITS == 4) { FLUTE_TRY(8, 4, 2, 4, 2); }
      if constexpr (BITS == 2) {
        FLUTE_TRY(8, 4, 2, 4, 3);
        FLUTE_TRY(8, 2, 2, 8, 2);  // (two-unit stages: 8 warps measured 6 % faster than 4)
      }
      FLUTE_TRY(8, 2, 2, 4, 2);
      break;
    case 16:
      if constexpr (BITS == 3) { FLUTE_TRY(16, 4, 2, 4, 3); }
      if constexpr (BITS != 4) { FLUTE_TRY(16, 2, 2, 4, 3); }
      // two-unit stages even when only two fit (W4 4096^2 M=16 6.50 -> 6.36 us,
      // W3 14336x4096 M=16 13.69 -> 12.64 us)
      FLUTE_TRY(16, 2, 2, 4, 2);
      FLUTE_TRY(16, 1, 2, 4, 2);
      break;
    default:
      if constexpr (BITS != 4) {
        FLUTE_TRY(32, 2, 2, 4, 3);
        FLUTE_TRY(32, 2, 2, 4, 2);  // (two two-unit stages beat one-unit ones by ~1 %)
        FLUTE_TRY(32, 1, 2, 4, 3);
        // (big cluster receive buffers: the one-CTA-per-SM kernel below)
      }
      FLUTE_TRY(32, 2, 1, 8, 2);
      break;
  }
#undef FLUTE_TRY
  throw flutesim::InternalError("qgemm: no kernel configuration fits shared memory");
}

// Cluster split-K (one cluster of C CTAs per 64-column tile, k split C ways,
// DSMEM reduction) when the tile count T fills >= 3/4 of the SMs with
// T*C <= #SMs; returns C (1 = no split), or 0 for Stream-K.
// CTAs per SM the kernel for an m-row launch is built for (launch_bits).
int occ_for(int m, int bits) { return bm_for(std::min(m, 32)) <= 16 || bits != 4 ? 2 : 1; }

int cluster_for(long long tiles_n, int tiles_k, int m, int bits) {
  if (std::getenv("FLUTE_NO_CLUSTER")) return 0;
  if (const char* f = std::getenv("FLUTE_FORCE_CLUSTER")) {  // tests: force cluster size C
    const int c = std::atoi(f);
    if (c >= 1 && c <= 8 && c <= tiles_k) return c;
  }
  // capacity: all co-resident CTA slots (two per SM for the OCC = 2 kernels,
  // measured faster than leaving the second slot to the next launch)
  const int sms = props().sms * occ_for(m, bits);
  for (int c = 8; c >= 1; c /= 2) {
    if (c > tiles_k) continue;
    const long long g = tiles_n * c;
    if (g <= sms && 4 * g >= 3LL * sms) {
      // one whole tile per CTA with slots left over (e.g. N = 14336: 224 of
      // 296): at M <= 8 Stream-K over every slot balances the SMs better
      // (4096x14336 M=4 10.68 -> 10.30 us, M=1 neutral to -4 %; at M >= 16
      // its fixups cost more than the balance gains)
      if (c == 1 && g < sms && m <= 8) return 0;
      return c;
    }
  }
  return 0;
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

int max_workers(int m, int bits) {
  return props().sms * occ_for(m, bits);  // co-resident CTA slots
}

int default_workers(int m, int k, int n, int bits) {
  (void)m;
  (void)bits;
  const int tiles_k = (k + kUnitK - 1) / kUnitK;
  const long long tiles_n = (n + kUnitN - 1) / kUnitN;
  const int c = cluster_for(tiles_n, tiles_k, m, bits);
  if (c > 0) return static_cast<int>(tiles_n * c);
  const long long slots = max_workers(m, bits);
  if (tiles_k * tiles_n <= slots) return static_cast<int>(tiles_k * tiles_n);
  // Stream-K: prefer a worker count that splits every t tiles into exactly c
  // ranges (P = tiles * c / t, t <= 4) when one comes within 10 % of the slot
  // count — a regular split measured ~2 % faster than filling every slot
  // (4096x14336 M<=8: 280 workers, 10.0-10.1 us vs 10.1-10.3 at 296;
  // profiles/r2/streamk_workers_sweep_r2h.txt)
  long long best = 0;
  for (long long t = 2; t <= 4; ++t)
    for (long long cc = t + 1; tiles_n * cc / t <= slots; ++cc)
      if ((tiles_n * cc) % t == 0 && tiles_n * cc / t > best) best = tiles_n * cc / t;
  if (10 * best >= 9 * slots) return static_cast<int>(best);
  return static_cast<int>(slots);
}

void debug_times(unsigned long long* out, int workers) {
  if (!g_dbg) throw flutesim::InputError("FLUTE_DEBUG_TIMES not enabled");
  // slot i (launch i of the ring) at out + i * workers * kDbgPerCta
  FLUTE_CUDA(cudaDeviceSynchronize());
  for (int i = 0; i < g_dbg_slots; ++i)
    FLUTE_CUDA(cudaMemcpy(out + static_cast<size_t>(i) * workers * kDbgPerCta,
                          g_dbg + static_cast<size_t>(i) * g_dbg_cap * kDbgPerCta,
                          static_cast<size_t>(std::min(workers, g_dbg_cap)) * kDbgPerCta * 8,
                          cudaMemcpyDeviceToHost));
}

size_t workspace_bytes(int m, int workers) {
  const int bm = bm_for(std::min(m, 32));
  const size_t flag_bytes = (static_cast<size_t>(workers) + 2) * 4;
  const size_t flag_span = (flag_bytes + 255) / 256 * 256;
  return flag_span + static_cast<size_t>(workers) * (bm / 8) * 16 * 32 * 4;
}

double time_launches(const std::function<void()>& fn, int reps, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int l2 = 0, dev = 0;
  FLUTE_CUDA(cudaGetDevice(&dev));
  FLUTE_CUDA(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev));
  const size_t flush_bytes = static_cast<size_t>(std::max(l2, 1 << 20)) * 2;
  void* flush = nullptr;
  FLUTE_CUDA(cudaMalloc(&flush, flush_bytes));
  cudaEvent_t e0, e1;
  FLUTE_CUDA(cudaEventCreate(&e0));
  FLUTE_CUDA(cudaEventCreate(&e1));
  double total_ms = 0;
  for (int r = 0; r < reps; ++r) {
    FLUTE_CUDA(cudaMemsetAsync(flush, r & 0xFF, flush_bytes, st));
    FLUTE_CUDA(cudaEventRecord(e0, st));
    fn();
    FLUTE_CUDA(cudaEventRecord(e1, st));
    FLUTE_CUDA(cudaEventSynchronize(e1));
    float ms = 0;
    FLUTE_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    total_ms += ms;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(flush);
  return total_ms * 1e3 / reps;
}

std::vector<Decomp> decomp_candidates(int m, int k, int n, int bits) {
  std::vector<Decomp> out;
  const int tiles_k = (k + kUnitK - 1) / kUnitK;
  const long long tiles_n = (n + kUnitN - 1) / kUnitN;
  const int slots = max_workers(std::min(m, 32), bits);
  out.push_back({-1, 0});  // the heuristic's own choice
  for (int c = 1; c <= 8; c *= 2)
    if (c <= tiles_k && tiles_n * c <= slots && 2 * tiles_n * c >= slots) out.push_back({c, 0});
  for (const int w : {props().sms, slots})
    if (w <= tiles_k * tiles_n) out.push_back({0, w});
  return out;
}

size_t tc_call_part_bytes(int m, int k, int n) {
  return tc_enabled(m) ? tc_workspace_bytes(m, k, n, props().sms) : 0;
}

size_t call_workspace_bytes(int m, int k, int n, int workers) {
  // (sized for the larger co-residency of any bit width)
  const size_t mma = workspace_bytes(std::min(m, 32), workers > 0 ? workers : max_workers(std::min(m, 32), 3) * 4);
  return tc_enabled(m) ? std::max(mma, tc_workspace_bytes(m, k, n, props().sms)) : mma;
}

void qgemm(const GemmArgs& a) {
  if (a.m < 1) throw flutesim::ConfigError("qgemm: m must be >= 1");
  if (a.bits < 2 || a.bits > 4) throw flutesim::ConfigError("qgemm: bits must be 2, 3 or 4");
  // every entry point (flute_qgemm, flute_qgemm_peers, handles) lands here:
  // the group must be a power of two in [32, 256] (the kernel shifts by
  // log2(group)) — a zero or odd group would otherwise divide by zero or pick
  // the wrong scales
  if (a.group < 32 || a.group > 256 || (a.group & (a.group - 1)) != 0)
    throw flutesim::ConfigError("qgemm: group must be a power of two in [32, 256], got " +
                                std::to_string(a.group));
  if (a.k % 16 != 0 || a.n % 16 != 0 || a.k < 16 || a.n < 16)
    throw flutesim::ConfigError("qgemm: k and n must be positive multiples of 16");
  if (!a.x || !a.w || !a.scales || !a.vlut || !a.workspace || (a.n_peers == 0 && !a.y))
    throw flutesim::InputError("qgemm: null device pointer");
  if (a.n_peers < 0 || a.n_peers > kMaxPeers)
    throw flutesim::ConfigError("qgemm: n_peers must be in [0, 8]");
  if (a.n_peers > 0) {
    for (int i = 0; i < a.n_peers; ++i)
      if (!a.y_peers || !a.y_peers[i]) throw flutesim::InputError("qgemm: null peer output pointer");
    if (a.ycol0 < 0 || a.ldy < a.ycol0 + a.n)
      throw flutesim::ConfigError("qgemm: peer output needs ldy >= ycol0 + n");
  }
  const int kp = (a.k + kUnitK - 1) / kUnitK * kUnitK;
  const int np = (a.n + kUnitN - 1) / kUnitN * kUnitN;
  if (kp % a.group != 0) throw flutesim::ConfigError("qgemm: padded k not divisible by group");
  const int tiles_k = kp / kUnitK;
  const long long units = static_cast<long long>(tiles_k) * (np / kUnitN);
  // default: cluster split-K when the tile count suits it, else Stream-K over
  // min(units, #SMs) CTAs; an explicit worker count always means Stream-K
  int cluster = a.cluster >= 1   ? std::min(a.cluster, tiles_k)
                : a.cluster == 0 ? 0
                : a.workers > 0  ? 0
                                 : cluster_for(np / kUnitN, tiles_k, a.m, a.bits);
  if (a.cluster == 0 && a.workers <= 0) cluster = 0;
  int workers = cluster > 0 ? static_cast<int>(np / kUnitN) * cluster
                            : (a.workers > 0 ? a.workers : default_workers(a.m, a.k, a.n, a.bits));
  if (units * (static_cast<long long>(workers) + 1) >= (1LL << 31))
    throw flutesim::ConfigError("qgemm: units x workers exceeds the 32-bit Stream-K index range");
  if (cluster == 0 && !(a.n_peers == 0 && tc_enabled(a.m)) &&
      a.workspace_bytes < workspace_bytes(a.m, workers))
    throw flutesim::InputError("qgemm: workspace too small");
  const int gp = kp / a.group;
  if (a.n_peers == 0 && tc_enabled(a.m)) {
    // compute-bound regime: one tcgen05 launch over all rows
    if (a.tc_part)
      qgemm_tc(a, tiles_k, np / kUnitN, gp, props().sms, false, a.tc_part, a.tc_part_bytes);
    else
      qgemm_tc(a, tiles_k, np / kUnitN, gp, props().sms, true, a.workspace, a.workspace_bytes);
    return;
  }
  // M > 32: 32-row chunks, stream-ordered on one workspace.
  for (int r0 = 0; r0 < a.m; r0 += 32) {
    const int rows = std::min(32, a.m - r0);
    const void* x = static_cast<const uint8_t*>(a.x) + static_cast<size_t>(r0) * a.k * 2;
    void* y = a.n_peers > 0
                  ? static_cast<void*>(static_cast<uint8_t*>(a.y_peers[0]) + static_cast<size_t>(r0) * a.ldy * 2)
                  : static_cast<void*>(static_cast<uint8_t*>(a.y) + static_cast<size_t>(r0) * a.n * 2);
    switch (a.bits) {
      case 2: launch_bits<2>(a, rows, x, y, workers, units, tiles_k, gp, cluster); break;
      case 3: launch_bits<3>(a, rows, x, y, workers, units, tiles_k, gp, cluster); break;
      default: launch_bits<4>(a, rows, x, y, workers, units, tiles_k, gp, cluster); break;
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
  fill_lut<BITS, 256, kTableRows<BITS>>(lut, vlut, threadIdx.x);
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
    } else if constexpr (BITS == 2) {
      uint32_t hw[2] = {0u, 0u};
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int pp = 0; pp < 4; ++pp) hw[j >> 1] |= d[4 * j + pp] << (8 * pp + 4 * (j & 1));
      lb.w = make_uint2(hw[0], hw[1]);
    } else {
      uint32_t wa, wb, wc;
      pack_lane_w3(d, wa, wb, wc);
      lb.hi = make_uint2(wa, wb);
      lb.lo = wc;
    }
    const uint32_t s = scales[si];
    const uint32_t sw = s | (s << 16);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      uint32_t a[4];
      lut_dequant4(atom_index_bytes<BITS>(lb, j), static_cast<uint32_t>(lane) * 4u, lut, sw, a);
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
  const int lut_bytes = kTableRows<4> * kLutRowBytes;
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

// ---------------------------------------------------------------------------
// host-buffer batches: copies in on one stream, GEMMs on the caller's stream,
// copies out on a third, chained by events, so item i's H2D and item i-1's
// D2H overlap the GEMMs.  Staging comes from a per-thread, per-device arena.
// ---------------------------------------------------------------------------

namespace {
struct BatchCtx {
  int dev = -1;
  cudaStream_t h2d = nullptr, d2h = nullptr;
  std::vector<cudaEvent_t> in_ready, out_ready;
  void* arena = nullptr;
  size_t arena_bytes = 0;

  void init(int d) {
    dev = d;
    FLUTE_CUDA(cudaStreamCreateWithFlags(&h2d, cudaStreamNonBlocking));
    FLUTE_CUDA(cudaStreamCreateWithFlags(&d2h, cudaStreamNonBlocking));
  }
  void events(size_t count) {
    while (in_ready.size() < count) {
      cudaEvent_t a, b;
      FLUTE_CUDA(cudaEventCreateWithFlags(&a, cudaEventDisableTiming));
      FLUTE_CUDA(cudaEventCreateWithFlags(&b, cudaEventDisableTiming));
      in_ready.push_back(a);
      out_ready.push_back(b);
    }
  }
  void* staging(size_t bytes) {
    if (bytes > arena_bytes) {
      if (arena) FLUTE_CUDA(cudaFree(arena));
      arena = nullptr;
      FLUTE_CUDA(cudaMalloc(&arena, bytes));
      arena_bytes = bytes;
    }
    return arena;
  }
};
}  // namespace

namespace {
// Enqueue the batch: copies in on h2d, GEMMs on st, copies out on d2h.  In
// capture mode there is no event query (illegal while capturing): inputs are
// waited for in doubling groups; in eager mode an input already resident is
// not waited for at all.
void enqueue_batch(const std::vector<HostBatchItem>& items, uint8_t* base,
                   const std::vector<size_t>& xo, const std::vector<size_t>& yo, cudaStream_t st,
                   cudaStream_t h2d, cudaStream_t d2h, cudaEvent_t start,
                   const std::vector<cudaEvent_t>& in_ready,
                   const std::vector<cudaEvent_t>& out_ready, bool capturing) {
  // Every cross-stream dependency on the GEMM stream costs two consecutive
  // GEMMs their programmatic-launch overlap, and every copy ~4 us of fixed
  // cost, so copies are grouped: inputs in groups growing from the front
  // ([0,2), [2,4), [4,8), ...: the first GEMM starts early, later inputs are
  // far ahead of the GEMMs — an M <= 32 input is <= 1 MB), outputs in groups
  // shrinking towards the back (..., [n-4,n-2), [n-2,n-1), [n-1,n): little is
  // left to copy after the last GEMM).  A group's copies are merged where its
  // items' host buffers are adjacent (a step's inputs / outputs allocated back
  // to back, as bench.py does); the staging layout keeps the device side
  // adjacent.  FLUTE_BATCH_WAIT_EACH=1: one item per group.
  static const bool each = std::getenv("FLUTE_BATCH_WAIT_EACH") != nullptr;
  const size_t n = items.size();
  std::vector<char> in_start(n + 1, 0), out_end(n + 1, 0);
  for (size_t b = 0; b < n; b = each ? b + 1 : std::max<size_t>(2, 2 * b)) in_start[b] = 1;
  out_end[n] = 1;  // output groups end at n, n-1, n-2, n-4, ... (sizes 1, 1, 2, 4, ...)
  for (size_t k = 1; k < n; k = each ? k + 1 : 2 * k) out_end[n - k] = 1;
  auto copy_range = [&](size_t a, size_t b, bool in) {
    for (size_t i = a; i < b;) {
      const uint8_t* h = static_cast<const uint8_t*>(in ? items[i].x_host : items[i].y_host);
      uint8_t* d = base + (in ? xo[i] : yo[i]);
      size_t bytes = in ? items[i].x_bytes : items[i].y_bytes;
      size_t j = i + 1;
      for (; j < b; ++j) {
        const uint8_t* hj = static_cast<const uint8_t*>(in ? items[j].x_host : items[j].y_host);
        if (hj != h + bytes || base + (in ? xo[j] : yo[j]) != d + bytes) break;
        bytes += in ? items[j].x_bytes : items[j].y_bytes;
      }
      if (in)
        FLUTE_CUDA(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, h2d));
      else
        FLUTE_CUDA(cudaMemcpyAsync(const_cast<uint8_t*>(h), d, bytes, cudaMemcpyDeviceToHost, d2h));
      i = j;
    }
  };
  FLUTE_CUDA(cudaEventRecord(start, st));
  FLUTE_CUDA(cudaStreamWaitEvent(h2d, start, 0));
  std::vector<size_t> in_ev(n, 0);  // input group event of each group start
  size_t ev = 0;
  for (size_t a = 0; a < n;) {
    size_t b = a + 1;
    while (b < n && !in_start[b]) ++b;
    copy_range(a, b, true);
    FLUTE_CUDA(cudaEventRecord(in_ready[ev], h2d));
    in_ev[a] = ev++;
    a = b;
  }
  size_t oev = 0, out_a = 0;
  for (size_t i = 0; i < n; ++i) {
    if (in_start[i] && (capturing || cudaEventQuery(in_ready[in_ev[i]]) != cudaSuccess))
      FLUTE_CUDA(cudaStreamWaitEvent(st, in_ready[in_ev[i]], 0));
    items[i].gemm(base + xo[i], base + yo[i], st);
    if (out_end[i + 1]) {
      FLUTE_CUDA(cudaEventRecord(out_ready[oev], st));
      FLUTE_CUDA(cudaStreamWaitEvent(d2h, out_ready[oev], 0));
      ++oev;
      copy_range(out_a, i + 1, false);
      out_a = i + 1;
    }
  }
}

// Staging: all inputs back to back, then all outputs (each 256-byte aligned),
// so items adjacent in host memory are adjacent on the device too.
size_t batch_layout(const std::vector<HostBatchItem>& items, std::vector<size_t>& xo,
                    std::vector<size_t>& yo) {
  xo.resize(items.size());
  yo.resize(items.size());
  size_t total = 0;
  for (size_t i = 0; i < items.size(); ++i) {
    xo[i] = total;
    total += (items[i].x_bytes + 255) / 256 * 256;
  }
  for (size_t i = 0; i < items.size(); ++i) {
    yo[i] = total;
    total += (items[i].y_bytes + 255) / 256 * 256;
  }
  return total;
}
}  // namespace

struct HostBatchGraph {
  void* arena = nullptr;
  cudaStream_t cap = nullptr, h2d = nullptr, d2h = nullptr;
  std::vector<cudaEvent_t> events;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
};

void host_batch_free(HostBatchGraph* g) {
  if (!g) return;
  if (g->exec) cudaGraphExecDestroy(g->exec);
  if (g->graph) cudaGraphDestroy(g->graph);
  for (cudaEvent_t e : g->events) cudaEventDestroy(e);
  if (g->cap) cudaStreamDestroy(g->cap);
  if (g->h2d) cudaStreamDestroy(g->h2d);
  if (g->d2h) cudaStreamDestroy(g->d2h);
  if (g->arena) cudaFree(g->arena);
  delete g;
}

HostBatchGraph* host_batch_capture(const std::vector<HostBatchItem>& items) {
  auto* g = new HostBatchGraph();
  try {
    for (const auto& it : items)
      if (it.prepare) it.prepare();  // workspace growth is not capturable
    std::vector<size_t> xo, yo;
    const size_t total = batch_layout(items, xo, yo);
    FLUTE_CUDA(cudaMalloc(&g->arena, total ? total : 256));
    FLUTE_CUDA(cudaStreamCreateWithFlags(&g->cap, cudaStreamNonBlocking));
    FLUTE_CUDA(cudaStreamCreateWithFlags(&g->h2d, cudaStreamNonBlocking));
    FLUTE_CUDA(cudaStreamCreateWithFlags(&g->d2h, cudaStreamNonBlocking));
    const size_t n = items.size();
    g->events.resize(2 * n + 2);
    for (auto& e : g->events) FLUTE_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    std::vector<cudaEvent_t> in(g->events.begin(), g->events.begin() + n);
    std::vector<cudaEvent_t> out(g->events.begin() + n, g->events.begin() + 2 * n);
    FLUTE_CUDA(cudaStreamBeginCapture(g->cap, cudaStreamCaptureModeThreadLocal));
    try {
      enqueue_batch(items, static_cast<uint8_t*>(g->arena), xo, yo, g->cap, g->h2d, g->d2h,
                    g->events[2 * n], in, out, true);
      // join the copy-out stream back into the origin stream
      FLUTE_CUDA(cudaEventRecord(g->events[2 * n + 1], g->d2h));
      FLUTE_CUDA(cudaStreamWaitEvent(g->cap, g->events[2 * n + 1], 0));
    } catch (...) {
      cudaGraph_t junk = nullptr;
      cudaStreamEndCapture(g->cap, &junk);
      if (junk) cudaGraphDestroy(junk);
      throw;
    }
    FLUTE_CUDA(cudaStreamEndCapture(g->cap, &g->graph));
    FLUTE_CUDA(cudaGraphInstantiate(&g->exec, g->graph, 0));
  } catch (...) {
    host_batch_free(g);
    throw;
  }
  return g;
}

void host_batch_run(HostBatchGraph* g, void* stream) {
  const cudaStream_t st = static_cast<cudaStream_t>(stream);
  FLUTE_CUDA(cudaGraphLaunch(g->exec, st));
  FLUTE_CUDA(cudaStreamSynchronize(st));
}

void host_batch(const std::vector<HostBatchItem>& items, void* stream) {
  if (items.empty()) return;
  static thread_local std::vector<BatchCtx> ctxs;
  int dev = 0;
  FLUTE_CUDA(cudaGetDevice(&dev));
  if (static_cast<int>(ctxs.size()) <= dev) ctxs.resize(dev + 1);
  BatchCtx& c = ctxs[dev];
  if (c.dev < 0) c.init(dev);
  c.events(items.size() + 1);
  for (const auto& it : items)
    if (it.prepare) it.prepare();
  const cudaStream_t st = static_cast<cudaStream_t>(stream);
  std::vector<size_t> xo, yo;
  uint8_t* base = static_cast<uint8_t*>(c.staging(batch_layout(items, xo, yo)));
  try {
    enqueue_batch(items, base, xo, yo, st, c.h2d, c.d2h, c.in_ready[items.size()], c.in_ready,
                  c.out_ready, false);
  } catch (...) {
    // drain what was queued before the failure so the arena is free again
    cudaStreamSynchronize(c.h2d);
    cudaStreamSynchronize(st);
    cudaStreamSynchronize(c.d2h);
    throw;
  }
  FLUTE_CUDA(cudaStreamSynchronize(c.d2h));
}

}  // namespace flute_dev
