// Prototype / calibration (not part of the product): tcgen05 with the A
// operand in tensor memory ("TS" MMA) for the LUT-GEMM.
//  A. thread -> (TMEM lane, column) mapping of tcgen05.st 16x128b / 16x256b
//  B. tcgen05.mma kind::f16, A from TMEM (M = 64 and 128), B = X^T from shared
//     memory (K-major, 128B swizzle), D in TMEM — checked against the CPU
//  C. throughput: LUT dequant (W4 vLUT, 32 lane copies) + tcgen05.st vs
//     LUT dequant + mma.sync, cycles per 256-weight atom per SM
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/_build/ts_proto tools/ts_proto.cu
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                          \
  do {                                                                                 \
    cudaError_t e_ = (x);                                                              \
    if (e_ != cudaSuccess) {                                                           \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      exit(1);                                                                         \
    }                                                                                  \
  } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void tmem_alloc(uint32_t slot, uint32_t cols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(slot), "r"(cols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t t, uint32_t cols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(t), "r"(cols) : "memory");
}
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void st_16x128_x2(uint32_t t, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("tcgen05.st.sync.aligned.16x128b.x2.b32 [%0], {%1, %2, %3, %4};" ::"r"(t), "r"(a), "r"(b),
               "r"(c), "r"(d)
               : "memory");
}
__device__ __forceinline__ void st_16x256_x1(uint32_t t, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("tcgen05.st.sync.aligned.16x256b.x1.b32 [%0], {%1, %2, %3, %4};" ::"r"(t), "r"(a), "r"(b),
               "r"(c), "r"(d)
               : "memory");
}
__device__ __forceinline__ void st_16x128_x8(uint32_t t, const uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.16x128b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, "
      "%13, %14, %15, %16};" ::"r"(t),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
      "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
}
__device__ __forceinline__ void st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void ld_32x32_x8(uint32_t t, uint32_t (&v)[8]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
      : "r"(t));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok = 0;
  while (!ok) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
  }
}
__device__ __forceinline__ uint64_t desc_sw128(uint32_t addr) {
  return static_cast<uint64_t>((addr >> 4) & 0x3FFFu) | (static_cast<uint64_t>(1) << 16) |
         (static_cast<uint64_t>(1024 >> 4) << 32) | (static_cast<uint64_t>(1) << 46) |
         (static_cast<uint64_t>(2) << 61);
}
__host__ __device__ constexpr uint32_t idesc_f16(int M, int N) {
  return (1u << 4) | (static_cast<uint32_t>(N >> 3) << 17) | (static_cast<uint32_t>(M >> 4) << 24);
}
__device__ __forceinline__ void umma_ts(uint32_t d, uint32_t a, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void umma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
               : "memory");
}

// ---------------------------------------------------------------- A: layout
__global__ void probe_layout(int shape, uint32_t* out) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) tmem_alloc(smem_u32(&slot), 32);
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t t = slot;
  const uint32_t tw = t + (static_cast<uint32_t>(warp * 32) << 16);
  // zero the warp's 32 lanes x 8 columns first
  {
    uint32_t z[16] = {};
    st_16x128_x8(tw, z);
    st_16x128_x8(tw + (16u << 16), z);
  }
  st_wait();
  uint32_t r[4];
  for (int i = 0; i < 4; ++i) r[i] = 0x80000000u | (warp << 16) | (lane << 8) | i;
  if (shape == 0) st_16x128_x2(tw, r[0], r[1], r[2], r[3]);
  else st_16x256_x1(tw, r[0], r[1], r[2], r[3]);
  st_wait();
  uint32_t v[8];
  ld_32x32_x8(tw, v);
  for (int c = 0; c < 8; ++c) out[(warp * 32 + lane) * 8 + c] = v[c];
  fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(t, 32);
}

// ---------------------------------------------------------------- B: TS MMA
// A: M x 64 (f16, row = output column n), B: NB x 64 (f16, row = x row m);
// D = A * B^T (M x NB fp32).  A goes to TMEM as mma.sync-style fragments
// (thread (g,t) of the warp handling rows 16j..16j+15: regs (g,kp t), (g+8,kp t),
// (g,kp t+4), (g+8,kp t+4) per 16-k step) with 16x128b.x2 stores.
template <int M, int NB>
__global__ void ts_mma_test(const __half* A, const __half* B, float* D) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t bsm = smem_u32(sm);
  // B tile: NB rows x 128 B (64 k), SW128: chunk c of row r at r*128 + ((c ^ (r&7))<<4)
  for (int i = threadIdx.x; i < NB * 8; i += blockDim.x) {
    const int r = i >> 3, c = i & 7;
    const uint4 v = *reinterpret_cast<const uint4*>(B + r * 64 + c * 8);
    *reinterpret_cast<uint4*>(sm + r * 128 + ((c ^ (r & 7)) << 4)) = v;
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) tmem_alloc(smem_u32(&slot), 128);
  if (threadIdx.x == 0) {
    mbar_init(smem_u32(&bar), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t t = slot;
  const int g = lane >> 2, tq = lane & 3;
  // A columns [0, 32): 4 k-steps x 8 columns; D at column 64
  const int atoms_per_warp = M / 64;  // M=64: one 16-row atom per warp, M=128: two
  for (int aw = 0; aw < atoms_per_warp; ++aw) {
    // rows of this atom and their TMEM lane base
    int row0, lane0;
    if (M == 64) {
      row0 = 16 * warp;
      lane0 = 32 * warp;
    } else {
      row0 = 32 * warp + 16 * aw;
      lane0 = 32 * warp + 16 * aw;
    }
    for (int ks = 0; ks < 4; ++ks) {
      auto pk = [&](int r, int kp) {
        const __half lo = A[(row0 + r) * 64 + 16 * ks + 2 * kp];
        const __half hi = A[(row0 + r) * 64 + 16 * ks + 2 * kp + 1];
        return static_cast<uint32_t>(__half_as_ushort(lo)) | (static_cast<uint32_t>(__half_as_ushort(hi)) << 16);
      };
      st_16x128_x2(t + (static_cast<uint32_t>(lane0) << 16) + 8 * ks, pk(g, tq), pk(g + 8, tq), pk(g, tq + 4),
                   pk(g + 8, tq + 4));
    }
  }
  st_wait();
  fence_before();
  __syncthreads();
  fence_after();
  if (threadIdx.x == 0) {
    for (int ks = 0; ks < 4; ++ks)
      umma_ts(t + 64, t + 8 * ks, desc_sw128(bsm + 32 * ks), idesc_f16(M, NB), ks > 0);
    umma_commit(smem_u32(&bar));
  }
  mbar_wait(smem_u32(&bar), 0);
  fence_after();
  // D: M=128 -> row r at lane r; M=64 -> row 16q+i at lane 32q+i
  for (int c0 = 0; c0 < NB; c0 += 8) {
    uint32_t v[8];
    ld_32x32_x8(t + (static_cast<uint32_t>(warp * 32) << 16) + 64 + c0, v);
    int row = -1;
    if (M == 128) row = warp * 32 + lane;
    else if (lane < 16) row = 16 * warp + lane;
    if (row >= 0)
      for (int c = 0; c < 8; ++c) D[row * NB + c0 + c] = __uint_as_float(v[c]);
  }
  fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(t, 128);
}

// ---------------------------------------------------------------- C: throughput
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t s) {
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(s));
  return r;
}
__device__ __forceinline__ uint32_t lds32c(uint32_t a) {
  uint32_t v;
  asm("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ uint4 lds128v(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ uint32_t hmul2(uint32_t a, uint32_t b) {
  uint32_t r;
  asm("mul.rn.f16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}

// MODE 0: dequant + tcgen05.st (4 atoms per 16x128b.x8), MODE 1: dequant + mma.sync,
// MODE 2: dequant only (results folded into an xor), MODE 3: dequant without HMUL2 + tcgen05.st
template <int MODE>
__global__ void loop_tput(int iters, uint32_t* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t* w = reinterpret_cast<uint32_t*>(sm);
  for (int i = threadIdx.x; i < (65536 + 16384) / 4; i += blockDim.x) w[i] = i * 2654435761u;
  const uint32_t lut = smem_u32(sm);
  const uint32_t data = lut + 65536;
  if (MODE == 0 || MODE == 3) {
    if (warp == 0) tmem_alloc(smem_u32(&slot), 512);
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t t = slot;
  const uint32_t lane4 = lane * 4;
  const uint32_t sc = 0x3c003c00u;
  uint32_t x = 0;
  float acc[4] = {0, 0, 0, 0};
  const uint32_t tw = t + (static_cast<uint32_t>((warp & 3) * 32 + ((warp >> 2) & 1) * 16) << 16) +
                      ((warp >> 3) * 32);
  for (int it = 0; it < iters; ++it) {
    // 4 atoms per iteration (one LDS.128 of packed indices per lane)
    const uint4 pk = lds128v(data + ((it & 31) * 512) + lane * 16);
    uint32_t v[16];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint32_t ib = j == 0 ? pk.x : j == 1 ? pk.y : j == 2 ? pk.z : pk.w;
#pragma unroll
      for (int p = 0; p < 4; ++p) {
        const uint32_t e = lds32c(lut + prmt(ib, lane4, 0x5504u | (p << 4)));
        v[4 * j + p] = MODE == 3 ? e : hmul2(e, sc);
      }
    }
    if (MODE == 0 || MODE == 3) {
      st_16x128_x8(tw + ((it & 7) * 64), v);
    } else if (MODE == 1) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        asm volatile(
            "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
            "{%0,%1,%2,%3};"
            : "+f"(acc[0]), "+f"(acc[1]), "+f"(acc[2]), "+f"(acc[3])
            : "r"(v[4 * j]), "r"(v[4 * j + 1]), "r"(v[4 * j + 2]), "r"(v[4 * j + 3]), "r"(sc), "r"(sc));
      }
    } else {
#pragma unroll
      for (int i = 0; i < 16; ++i) x ^= v[i];
    }
  }
  if (MODE == 0 || MODE == 3) st_wait();
  if (x == 0x12345u || acc[0] == 1.2345f) out[0] = x;
  fence_before();
  __syncthreads();
  if ((MODE == 0 || MODE == 3) && warp == 0) tmem_dealloc(t, 512);
}

int main() {
  // ---- A
  uint32_t* d_out;
  CK(cudaMalloc(&d_out, 128 * 8 * 4));
  std::vector<uint32_t> h(128 * 8);
  for (int shape = 0; shape < 2; ++shape) {
    CK(cudaMemset(d_out, 0, 128 * 8 * 4));
    probe_layout<<<1, 128>>>(shape, d_out);
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(h.data(), d_out, h.size() * 4, cudaMemcpyDeviceToHost));
    printf("== %s: TMEM (lane, col) <- (warp, thread, reg) for warp 0\n",
           shape == 0 ? "16x128b.x2" : "16x256b.x1");
    for (int l = 0; l < 32; ++l) {
      printf("lane %2d:", l);
      for (int c = 0; c < 8; ++c) {
        const uint32_t v = h[l * 8 + c];
        if (v & 0x80000000u) printf(" t%02d.r%d", (v >> 8) & 0xff, v & 0xff);
        else printf("   ---- ");
      }
      printf("\n");
    }
  }
  // ---- B
  auto runB = [&](auto mtag, auto ntag) {
    constexpr int M = decltype(mtag)::value, NB = decltype(ntag)::value;
    std::vector<__half> a(M * 64), b(NB * 64);
    srand(7);
    for (auto& v : a) v = __float2half((rand() % 17 - 8) / 4.0f);
    for (auto& v : b) v = __float2half((rand() % 13 - 6) / 2.0f);
    __half *da, *db;
    float* dd;
    CK(cudaMalloc(&da, a.size() * 2));
    CK(cudaMalloc(&db, b.size() * 2));
    CK(cudaMalloc(&dd, M * NB * 4));
    CK(cudaMemcpy(da, a.data(), a.size() * 2, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(db, b.data(), b.size() * 2, cudaMemcpyHostToDevice));
    CK(cudaMemset(dd, 0, M * NB * 4));
    ts_mma_test<M, NB><<<1, 128, 32 * 1024>>>(da, db, dd);
    CK(cudaDeviceSynchronize());
    std::vector<float> d(M * NB);
    CK(cudaMemcpy(d.data(), dd, d.size() * 4, cudaMemcpyDeviceToHost));
    int bad = 0;
    for (int r = 0; r < M; ++r)
      for (int c = 0; c < NB; ++c) {
        float ref = 0;
        for (int k = 0; k < 64; ++k) ref += __half2float(a[r * 64 + k]) * __half2float(b[c * 64 + k]);
        if (fabsf(ref - d[r * NB + c]) > 1e-3f) {
          if (bad < 5) printf("  mismatch r=%d c=%d ref=%g got=%g\n", r, c, ref, d[r * NB + c]);
          ++bad;
        }
      }
    printf("== TS MMA M=%d N=%d: %s (%d mismatches)\n", M, NB, bad ? "FAIL" : "ok", bad);
  };
  runB(std::integral_constant<int, 64>{}, std::integral_constant<int, 8>{});
  runB(std::integral_constant<int, 64>{}, std::integral_constant<int, 16>{});
  runB(std::integral_constant<int, 128>{}, std::integral_constant<int, 16>{});
  runB(std::integral_constant<int, 128>{}, std::integral_constant<int, 32>{});
  // ---- C
  const int iters = 4096;
  auto tput = [&](auto kern, const char* name) {
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024));
    for (int warps : {4, 8, 12, 16}) {
      kern<<<148, warps * 32, 82 * 1024>>>(16, d_out);
      CK(cudaDeviceSynchronize());
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0);
      kern<<<148, warps * 32, 82 * 1024>>>(iters, d_out);
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double atoms_per_sm = static_cast<double>(iters) * 4 * warps;
      const double cyc = ms * 1e-3 * 1.965e9;
      printf("%-34s warps=%2d: %6.2f SM-cycles/atom (at 1.965 GHz), %.3f ms\n", name, warps,
             cyc / atoms_per_sm, ms);
    }
  };
  tput(loop_tput<0>, "LUT+HMUL2 -> tcgen05.st");
  tput(loop_tput<3>, "LUT (no HMUL2) -> tcgen05.st");
  tput(loop_tput<1>, "LUT+HMUL2 -> mma.sync");
  tput(loop_tput<2>, "LUT+HMUL2 only");
  return 0;
}
