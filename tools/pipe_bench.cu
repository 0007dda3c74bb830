// Calibration microbenchmark (not part of the product): per-SM throughput of
// the instruction classes the LUT-GEMM inner loop is made of, on sm_100a:
//   HMMA.16816.F32 (mma.sync m16n8k16, fp32 accumulate), HMMA.16816.F16,
//   LDS.32 lookups with the 32-copy vLUT address pattern, PRMT, HMUL2.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/_build/pipe_bench tools/pipe_bench.cu
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

template <int CHAINS>
__global__ void hmma_f32(int iters, float* out) {
  float d[CHAINS][4];
  for (int c = 0; c < CHAINS; ++c) for (int r = 0; r < 4; ++r) d[c][r] = 0.f;
  uint32_t a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 ^ 0x3c003c00u, b1 = b0 + 1;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+f"(d[c][0]), "+f"(d[c][1]), "+f"(d[c][2]), "+f"(d[c][3])
                   : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  float s = 0.f;
  for (int c = 0; c < CHAINS; ++c) for (int r = 0; r < 4; ++r) s += d[c][r];
  if (s == 1.2345f) out[0] = s;
}

template <int CHAINS>
__global__ void hmma_f16(int iters, float* out) {
  uint32_t d[CHAINS][2];
  for (int c = 0; c < CHAINS; ++c) d[c][0] = d[c][1] = 0u;
  uint32_t a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 ^ 0x3c003c00u, b1 = b0 + 1;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f16.f16.f16.f16 {%0,%1}, {%2,%3,%4,%5}, {%6,%7}, {%0,%1};"
                   : "+r"(d[c][0]), "+r"(d[c][1])
                   : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  uint32_t s = 0;
  for (int c = 0; c < CHAINS; ++c) s ^= d[c][0] ^ d[c][1];
  if (s == 12345u) out[0] = s;
}

// 32-copy vLUT lookups: address = (e << 8) | (lane << 2), e pseudo-random.
__global__ void lds_lut(int iters, float* out) {
  extern __shared__ uint32_t lut[];
  for (int i = threadIdx.x; i < 16384; i += blockDim.x) lut[i] = i;
  __syncthreads();
  const uint32_t base = static_cast<uint32_t>(__cvta_generic_to_shared(lut));
  uint32_t x = threadIdx.x * 2654435761u, acc = 0;
  const uint32_t lane4 = (threadIdx.x & 31) * 4;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      uint32_t off;
      asm("prmt.b32 %0, %1, %2, 0x5504;" : "=r"(off) : "r"(x >> (j * 2)), "r"(lane4));
      uint32_t v;
      asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(base + off));
      acc += v;
    }
    x = x * 1664525u + 1013904223u;
  }
  if (acc == 0x12345u) out[0] = acc;
}

// The LUT-GEMM inner loop in isolation: per iteration each warp loads 16 B of
// packed W4 indices + a scale word vector + an X fragment from shared memory,
// then dequantises ATOMS atoms (4 x PRMT->LDS->HMUL2) and issues HMMAs.
// VAR: 0 full, 1 no HMUL2, 2 no vLUT LDS (index bytes used as data), 3 no HMMA.
template <int VAR, int ATOMS>
__global__ void lut_mma_loop(int iters, float* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint32_t* w = reinterpret_cast<uint32_t*>(sm);
  for (int i = threadIdx.x; i < 65536 / 4 + 8192; i += blockDim.x) w[i] = i * 2654435761u;
  __syncthreads();
  const uint32_t lut = static_cast<uint32_t>(__cvta_generic_to_shared(sm));
  const uint32_t data = lut + 65536;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t lane4 = lane * 4;
  float acc[4][4] = {};
  uint32_t sink = 0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int h = 0; h < ATOMS / 4; ++h) {
      const uint32_t off = data + ((i * 8 + warp + h * 3) & 63) * 512;
      uint4 lb, sq;
      asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(lb.x), "=r"(lb.y), "=r"(lb.z), "=r"(lb.w) : "r"(off + lane * 16));
      asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(sq.x), "=r"(sq.y), "=r"(sq.z), "=r"(sq.w) : "r"(off + (lane >> 2) * 16));
      uint32_t b0, b1;
      asm volatile("ldmatrix.sync.aligned.m8n8.x2.shared.b16 {%0, %1}, [%2];" : "=r"(b0), "=r"(b1) : "r"(off + (lane & 15) * 16));
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t idx = j == 0 ? lb.x : j == 1 ? lb.y : j == 2 ? lb.z : lb.w;
        const uint32_t scw = j == 0 ? sq.x : j == 1 ? sq.y : j == 2 ? sq.z : sq.w;
        const __half2 s2 = *reinterpret_cast<const __half2*>(&scw);
        uint32_t a[4];
#pragma unroll
        for (int pp = 0; pp < 4; ++pp) {
          uint32_t o;
          asm("prmt.b32 %0, %1, %2, %3;" : "=r"(o) : "r"(idx), "r"(lane4), "r"(0x5504u | (pp << 4)));
          uint32_t v;
          if (VAR == 2) v = o;
          else asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(lut + o));
          if (VAR == 1) {
            a[pp] = v;
          } else {
            const __half2 r = __hmul2(*reinterpret_cast<const __half2*>(&v), (pp & 1) ? __high2half2(s2) : __low2half2(s2));
            a[pp] = *reinterpret_cast<const uint32_t*>(&r);
          }
        }
        if (VAR == 3) {
          sink ^= a[0] ^ a[1] ^ a[2] ^ a[3] ^ b0 ^ b1;
        } else {
          asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                       : "+f"(acc[j][0]), "+f"(acc[j][1]), "+f"(acc[j][2]), "+f"(acc[j][3])
                       : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
        }
      }
    }
  }
  float s = 0.f;
  for (int j = 0; j < 4; ++j) for (int r = 0; r < 4; ++r) s += acc[j][r];
  if (s == 1.2345f || sink == 0x1234567u) out[0] = s;
}

// The same loop for MT 8-row m-tiles of X per atom (M = 8*MT rows): each atom's
// dequantised A feeds MT HMMAs with different B fragments (the M = 16 / 32
// kernels), 4*MT accumulators per atom column.
template <int MT>
__global__ void lut_mma_loop_mt(int iters, float* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint32_t* w = reinterpret_cast<uint32_t*>(sm);
  for (int i = threadIdx.x; i < 65536 / 4 + 8192; i += blockDim.x) w[i] = i * 2654435761u;
  __syncthreads();
  const uint32_t lut = static_cast<uint32_t>(__cvta_generic_to_shared(sm));
  const uint32_t data = lut + 65536;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t lane4 = lane * 4;
  float acc[MT][4][4] = {};
  for (int i = 0; i < iters; ++i) {
    const uint32_t off = data + ((i * 8 + warp) & 63) * 512;
    uint4 lb, sq;
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(lb.x), "=r"(lb.y), "=r"(lb.z), "=r"(lb.w) : "r"(off + lane * 16));
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(sq.x), "=r"(sq.y), "=r"(sq.z), "=r"(sq.w) : "r"(off + (lane >> 2) * 16));
    uint32_t b[MT][2];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
      asm volatile("ldmatrix.sync.aligned.m8n8.x2.shared.b16 {%0, %1}, [%2];" : "=r"(b[mt][0]), "=r"(b[mt][1]) : "r"(off + ((lane + 16 * mt) & 31) * 16));
    uint32_t v[4][4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint32_t idx = j == 0 ? lb.x : j == 1 ? lb.y : j == 2 ? lb.z : lb.w;
#pragma unroll
      for (int pp = 0; pp < 4; ++pp) {
        uint32_t o;
        asm("prmt.b32 %0, %1, %2, %3;" : "=r"(o) : "r"(idx), "r"(lane4), "r"(0x5504u | (pp << 4)));
        asm("ld.shared.u32 %0, [%1];" : "=r"(v[j][pp]) : "r"(lut + o));
      }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint32_t scw = j == 0 ? sq.x : j == 1 ? sq.y : j == 2 ? sq.z : sq.w;
      const __half2 s2 = *reinterpret_cast<const __half2*>(&scw);
      uint32_t a[4];
#pragma unroll
      for (int pp = 0; pp < 4; ++pp) {
        const __half2 r = __hmul2(*reinterpret_cast<const __half2*>(&v[j][pp]), (pp & 1) ? __high2half2(s2) : __low2half2(s2));
        a[pp] = *reinterpret_cast<const uint32_t*>(&r);
      }
#pragma unroll
      for (int mt = 0; mt < MT; ++mt)
        asm("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
            : "+f"(acc[mt][j][0]), "+f"(acc[mt][j][1]), "+f"(acc[mt][j][2]), "+f"(acc[mt][j][3])
            : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[mt][0]), "r"(b[mt][1]));
    }
  }
  float s = 0.f;
  for (int mt = 0; mt < MT; ++mt) for (int j = 0; j < 4; ++j) for (int r = 0; r < 4; ++r) s += acc[mt][j][r];
  if (s == 1.2345f) out[0] = s;
}

// mbarrier costs: (a) try_wait on an already-completed phase, (b) a
// producer/consumer ping-pong through a ring of S barriers (no data).
__global__ void mbar_latency(int iters, float* out) {
  __shared__ __align__(8) unsigned long long bars[128];
  const uint32_t b0 = static_cast<uint32_t>(__cvta_generic_to_shared(bars));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 32; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b0 + 8 * i), "r"(1) : "memory");
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b0 + 256 + 8 * i), "r"(4) : "memory");
    }
    for (int i = 0; i < 8; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b0 + 512 + 8 * i), "r"(1) : "memory");
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b0 + 576 + 8 * i), "r"(4) : "memory");
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  long long t0 = clock64();
  if (blockIdx.x == 0 && iters < 0) {
  }
  // (a) completed-phase try_wait: complete phase 0 of bar 40 then wait on it repeatedly
  if (warp == 0) {
    const uint32_t bar = b0 + 8 * 40;
    if (lane == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(1) : "memory");
      asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(bar) : "memory");
    }
    __syncwarp();
    t0 = clock64();
    uint32_t okc = 0;
    for (int i = 0; i < iters; ++i) {
      uint32_t ok;
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                   : "=r"(ok) : "r"(bar), "r"(0u) : "memory");
      okc += ok;
    }
    long long t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) printf("  try_wait on a completed phase: %.1f cycles/call (ok=%u)\n", double(t1 - t0) / iters, okc);
  }
  __syncthreads();
  // (b) ring ping-pong: warp 0 = producer (waits empty, arrives full), warps 1..4 consumers
  const int S = out ? 4 : 4;
  if (warp == 0) {
    t0 = clock64();
    for (int i = 0, s = 0, ph = 0; i < iters; ++i) {
      if (i >= S) {
        uint32_t ok = 0;
        while (!ok) asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                                 : "=r"(ok) : "r"(b0 + 256 + 8 * s), "r"(ph ^ 1u) : "memory");
      }
      if (lane == 0) asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(b0 + 8 * s) : "memory");
      if (++s == S) { s = 0; ph ^= 1; }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) printf("  ring of %d, 1 producer + 4 consumer warps: %.1f cycles/stage\n", S, double(t1 - t0) / iters);
  } else if (warp <= 4) {
    for (int i = 0, s = 0, ph = 0; i < iters; ++i) {
      uint32_t ok = 0;
      while (!ok) asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                               : "=r"(ok) : "r"(b0 + 8 * s), "r"(ph) : "memory");
      __syncwarp();
      if (lane == 0) asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(b0 + 256 + 8 * s) : "memory");
      if (++s == S) { s = 0; ph ^= 1; }
    }
  }
  __syncthreads();
  // (b) ring ping-pong: warp 0 = producer (waits empty, arrives full), warps 1..4 consumers
  const int S3 = 4;
  if (warp == 0) {
    t0 = clock64();
    for (int i = 0, s = 0, ph = 0; i < iters; ++i) {
      if (i >= S3) {
        uint32_t ok = 0;
        while (!ok) asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                                 : "=r"(ok) : "r"(b0 + 576 + 8 * s), "r"(ph ^ 1u) : "memory");
      }
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(b0 + 512 + 8 * s) : "memory");
      if (++s == S3) { s = 0; ph ^= 1; }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) printf("  ring of %d, sink-form arrive: %.1f cycles/stage\n", S3, double(t1 - t0) / iters);
  } else if (warp <= 4) {
    for (int i = 0, s = 0, ph = 0; i < iters; ++i) {
      uint32_t ok = 0;
      while (!ok) asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                               : "=r"(ok) : "r"(b0 + 512 + 8 * s), "r"(ph) : "memory");
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(b0 + 576 + 8 * s) : "memory");
      if (++s == S3) { s = 0; ph ^= 1; }
    }
  }
  __syncthreads();
  // (b) ring ping-pong: warp 0 = producer (waits empty, arrives full), warps 1..4 consumers
  const int S2 = 4;
  if (warp == 0) {
    t0 = clock64();
    for (int i = 0, s = 0, ph = 0; i < iters; ++i) {
      if (i >= S2) {
        uint32_t ok = 0;
        while (!ok) asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                                 : "=r"(ok) : "r"(b0 + 256 + 8 * (s + 16)), "r"(ph ^ 1u) : "memory");
      }
      if (lane == 0) asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(b0 + 8 * (s + 16)) : "memory");
      if (++s == S2) { s = 0; ph ^= 1; }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) printf("  ring of %d (test_wait spin): %.1f cycles/stage\n", S2, double(t1 - t0) / iters);
  } else if (warp <= 4) {
    for (int i = 0, s = 0, ph = 0; i < iters; ++i) {
      uint32_t ok = 0;
      while (!ok) asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                               : "=r"(ok) : "r"(b0 + 8 * (s + 16)), "r"(ph) : "memory");
      __syncwarp();
      if (lane == 0) asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(b0 + 256 + 8 * (s + 16)) : "memory");
      if (++s == S) { s = 0; ph ^= 1; }
    }
  }
  if (iters == -7) out[0] = 1.f;
}

// Per-op issue cost of mbarrier.arrive.expect_tx and cp.async.bulk from one
// thread (barriers re-initialised each round so phases always complete).
__global__ void arrive_cost(const uint8_t* src, float* out) {
  __shared__ __align__(8) unsigned long long bars[16];
  __shared__ __align__(128) uint8_t buf[16 * 1024];
  const uint32_t b0 = static_cast<uint32_t>(__cvta_generic_to_shared(bars));
  const uint32_t d0 = static_cast<uint32_t>(__cvta_generic_to_shared(buf));
  if (threadIdx.x != 0) return;
  long long t_init = 0, t_arr = 0, t_tx = 0, t_bulk = 0;
  for (int round = 0; round < 20; ++round) {
    long long t0 = clock64();
    for (int i = 0; i < 16; ++i)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b0 + 8 * i), "r"(1) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    long long t1 = clock64();
    for (int i = 0; i < 8; ++i)
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(b0 + 8 * i) : "memory");
    long long t2 = clock64();
    for (int i = 8; i < 16; ++i)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b0 + 8 * i), "r"(1024u) : "memory");
    long long t3 = clock64();
    for (int i = 8; i < 16; ++i)
      asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(d0 + (i - 8) * 1024),
                   "l"(src + (round * 16 + i) * 4096), "r"(1024u), "r"(b0 + 8 * i) : "memory");
    long long t4 = clock64();
    for (int i = 8; i < 16; ++i) {
      uint32_t ok = 0;
      while (!ok) asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(b0 + 8 * i), "r"(0u) : "memory");
    }
    if (round > 0) { t_init += t1 - t0; t_arr += t2 - t1; t_tx += t3 - t2; t_bulk += t4 - t3; }
  }
  printf("  per op (cycles): mbarrier.init %.1f | arrive %.1f | arrive.expect_tx %.1f | cp.async.bulk 1KB issue %.1f\n",
         t_init / (19.0 * 16), t_arr / (19.0 * 8), t_tx / (19.0 * 8), t_bulk / (19.0 * 8));
  out[0] = 0.f;
}

template <class K>
void run(const char* name, K kern, int threads, size_t smem, double work_per_thread_iter, const char* unit, int iters) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out;
  cudaMalloc(&out, 4);
  if (smem) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  kern<<<sms, threads, smem>>>(iters, out);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  kern<<<sms, threads, smem>>>(iters, out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double tot = work_per_thread_iter * threads / 32.0 * iters * sms;
  printf("%-28s threads %4d: %10.2f %s  (%.2f per SM per ns)\n", name, threads, tot / (ms * 1e-3) / 1e12,
         unit, tot / sms / (ms * 1e6));
  cudaError_t e = cudaGetLastError();
  if (e) printf("  error %s\n", cudaGetErrorString(e));
}

int main() {
  const int it = 20000;
  {
    float* o;
    cudaMalloc(&o, 4);
    mbar_latency<<<1, 160>>>(10000, o);
    cudaDeviceSynchronize();
    uint8_t* src;
    cudaMalloc(&src, 4 << 20);
    arrive_cost<<<1, 32>>>(src, o);
    cudaDeviceSynchronize();
  }
  const size_t sm = 65536 + 32768 + 1024;
  if (getenv("MT_ONLY")) {
    for (int th : {256, 384, 512}) {
      run("MT=1 (M<=8)", lut_mma_loop_mt<1>, th, sm, 4.0, "T atoms/s", it / 4);
      run("MT=2 (M=16)", lut_mma_loop_mt<2>, th, sm, 4.0, "T atoms/s", it / 4);
      run("MT=4 (M=32)", lut_mma_loop_mt<4>, th, sm, 4.0, "T atoms/s", it / 4);
    }
    return 0;
  }
  for (int th : {256, 512}) {
    run("full, 4 atoms/iter", lut_mma_loop<0, 4>, th, sm, 4.0, "T atoms/s", it / 4);
    run("full, 8 atoms/iter", lut_mma_loop<0, 8>, th, sm, 8.0, "T atoms/s", it / 8);
    run("full, 16 atoms/iter", lut_mma_loop<0, 16>, th, sm, 16.0, "T atoms/s", it / 16);
    run("no HMUL2, 8", lut_mma_loop<1, 8>, th, sm, 8.0, "T atoms/s", it / 8);
    run("no vLUT LDS, 8", lut_mma_loop<2, 8>, th, sm, 8.0, "T atoms/s", it / 8);
    run("no HMMA, 8", lut_mma_loop<3, 8>, th, sm, 8.0, "T atoms/s", it / 8);
  }
  return 0;
  for (int th : {128, 256, 512, 1024}) {
    run("hmma f32acc 1 chain", hmma_f32<1>, th, 0, 4096.0, "TFLOP/s", it);
    run("hmma f32acc 4 chains", hmma_f32<4>, th, 0, 4 * 4096.0, "TFLOP/s", it);
    run("hmma f16acc 4 chains", hmma_f16<4>, th, 0, 4 * 4096.0, "TFLOP/s", it);
    run("lds lut (warp-instr)", lds_lut, th, 65536, 8.0, "T warp-LDS/s", it);
  }
  return 0;
}
