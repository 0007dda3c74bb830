// Calibration microbenchmark (not part of the product): how fast can one
// producer thread per CTA stream a contiguous HBM range into a shared-memory
// ring with 1-D bulk async copies (cp.async.bulk, UBLKCP), with consumer warps
// that only wait on the full barrier and release the slot?
//
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/_build/tma_stream_bench tools/tma_stream_bench.cu
// run:   tools/_build/tma_stream_bench   (prints GB/s per configuration)
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(bar)
               : "memory");
}
__device__ __forceinline__ void mbar_expect(uint32_t bar, uint32_t bytes) {
  asm volatile(
      "{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(bar),
      "r"(bytes)
      : "memory");
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
__device__ __forceinline__ void bulk(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}

// ncons consumer warps + 1 producer warp; chunk = bytes per stage; S stages;
// `copies` bulk ops per stage (chunk split evenly).
__global__ void stream_kernel(const uint8_t* src, size_t per_cta, int S, uint32_t chunk, int copies,
                              int ncons, unsigned long long* sink) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t base = smem_u32(smem);
  const uint32_t bars = base + S * chunk;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(bars + 8 * s, 1);
      mbar_init(bars + 8 * (S + s), ncons);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint8_t* my = src + per_cta * blockIdx.x;
  const int n = static_cast<int>(per_cta / chunk);
  if (warp == ncons) {
    if (lane == 0) {
      const uint32_t part = chunk / copies;
      for (int it = 0, s = 0, ph = 0; it < n; ++it) {
        if (it >= S) mbar_wait(bars + 8 * (S + s), ph ^ 1);
        mbar_expect(bars + 8 * s, chunk);
        for (int c = 0; c < copies; ++c)
          bulk(base + s * chunk + c * part, my + static_cast<size_t>(it) * chunk + c * part, part,
               bars + 8 * s);
        if (++s == S) { s = 0; ph ^= 1; }
      }
    }
  } else {
    unsigned long long acc = 0;
    for (int it = 0, s = 0, ph = 0; it < n; ++it) {
      mbar_wait(bars + 8 * s, ph);
      uint32_t v;
      asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(base + s * chunk + (warp * 32 + lane) * 4));
      acc += v;
      __syncwarp();
      if (lane == 0) mbar_arrive(bars + 8 * (S + s));
      if (++s == S) { s = 0; ph ^= 1; }
    }
    if (acc == 0x1234567) sink[0] = acc;
  }
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t total = size_t(1) << 30;  // 1 GiB source, well beyond L2
  uint8_t* src;
  unsigned long long* sink;
  cudaMalloc(&src, total);
  cudaMalloc(&sink, 8);
  cudaMemset(src, 1, total);
  struct Cfg { int ctas_per_sm, S; uint32_t chunk; int copies, ncons; };
  std::vector<Cfg> cfgs = {
      {1, 4, 16384, 1, 8},  {1, 8, 16384, 1, 8},  {1, 12, 16384, 1, 8}, {1, 8, 8192, 1, 8},
      {1, 16, 8192, 1, 8},  {1, 24, 8192, 1, 8},  {1, 16, 4096, 1, 8},  {1, 32, 4096, 1, 8},
      {1, 6, 32768, 1, 8},  {1, 8, 16384, 4, 8},  {2, 6, 16384, 1, 8},  {2, 12, 8192, 1, 8},
      {4, 6, 8192, 1, 4},   {1, 8, 16384, 1, 1},  {1, 8, 16384, 1, 16},
  };
  printf("ctas/sm stages chunk copies cons  |  GB/s (1 GiB stream)   |  GB/s (23 MB per launch) | GB/s (8.5 MB per launch)\n");
  for (const Cfg& c : cfgs) {
    const int grid = sms * c.ctas_per_sm;
    const size_t smem = size_t(c.S) * c.chunk + 16 * c.S + 64;
    cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    double gbs[3];
    for (int mode = 0; mode < 3; ++mode) {
      const size_t bytes = mode == 0 ? total : mode == 1 ? size_t(23) << 20 : size_t(17) << 19;
      size_t per_cta = bytes / grid / c.chunk * c.chunk;
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      const int reps = mode == 0 ? 5 : 40;
      // mode 1 rotates through the GiB so each launch reads cold data
      for (int w = 0; w < 3; ++w)
        stream_kernel<<<grid, 32 * (c.ncons + 1), smem>>>(src, per_cta, c.S, c.chunk, c.copies, c.ncons, sink);
      cudaEventRecord(e0);
      for (int r = 0; r < reps; ++r) {
        const uint8_t* s = mode == 0 ? src : src + (size_t(r % 40) * (size_t(24) << 20)) % (total - bytes);
        stream_kernel<<<grid, 32 * (c.ncons + 1), smem>>>(s, per_cta, c.S, c.chunk, c.copies, c.ncons, sink);
      }
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      gbs[mode] = double(per_cta) * grid * reps / (ms * 1e-3) / 1e9;
      cudaError_t err = cudaGetLastError();
      if (err != cudaSuccess) printf("error %s\n", cudaGetErrorString(err));
    }
    printf("%7d %6d %6u %6d %4d  |  %8.0f               |  %8.0f  |  %8.0f\n", c.ctas_per_sm, c.S,
           c.chunk, c.copies, c.ncons, gbs[0], gbs[1], gbs[2]);
  }
  return 0;
}
