// Calibration microbenchmark (not part of the product): back-to-back launches
// of a bulk-copy streaming kernel over a small per-launch footprint (8.5 / 23
// MB, cold in HBM), with and without programmatic dependent launch (PDL), and
// with shared memory small enough for a CTA of the next launch to co-reside.
// The first `pre` stages are issued BEFORE griddepcontrol.wait (as the GEMM
// prefetches weights), the rest after.
//
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/_build/pdl_stream_bench tools/pdl_stream_bench.cu
// run:   tools/_build/pdl_stream_bench
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


__global__ void stream_kernel(const uint8_t* src, size_t per_cta, int S, uint32_t chunk, int ncons,
                              int pdl, unsigned long long* sink) {
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
  if (pdl) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const uint8_t* my = src + per_cta * blockIdx.x;
  const int n = static_cast<int>(per_cta / chunk);
  if (warp == ncons) {
    if (lane == 0) {
      for (int it = 0, s = 0, ph = 0; it < n; ++it) {
        if (it == S && pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
        if (it >= S) mbar_wait(bars + 8 * (S + s), ph ^ 1);
        mbar_expect(bars + 8 * s, chunk);
        bulk(base + s * chunk, my + static_cast<size_t>(it) * chunk, chunk, bars + 8 * s);
        if (++s == S) { s = 0; ph ^= 1; }
      }
      if (n <= S && pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
    }
  } else {
    if (pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
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
  const size_t total = size_t(1) << 30;
  uint8_t* src;
  unsigned long long* sink;
  cudaMalloc(&src, total);
  cudaMalloc(&sink, 8);
  cudaMemset(src, 1, total);
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  struct Cfg { int S; uint32_t chunk; int ncons; };
  std::vector<Cfg> cfgs = {{12, 16384, 8}, {6, 16384, 8}, {12, 8192, 8}, {6, 8192, 8}, {24, 4096, 8},
                           {12, 4096, 8}, {3, 32768, 8}};
  printf("stages chunk smemKB | MB/launch | GB/s eager | eager+PDL | graph | graph+PDL\n");
  for (const Cfg& c : cfgs) {
    const size_t smem = size_t(c.S) * c.chunk + 16 * c.S + 64;
    cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    for (size_t bytes : {size_t(17) << 19, size_t(23) << 20}) {
      size_t per_cta = bytes / sms / c.chunk * c.chunk;
      double gbs[4];
      for (int mode = 0; mode < 4; ++mode) {
        const int pdl = mode & 1, graph = mode >> 1;
        const int reps = 40;
        auto launch_all = [&]() {
          for (int r = 0; r < reps; ++r) {
            const uint8_t* s = src + (size_t(r % 40) * (size_t(24) << 20)) % (total - bytes);
            cudaLaunchConfig_t cfg{};
            cfg.gridDim = dim3(sms);
            cfg.blockDim = dim3(32 * (c.ncons + 1));
            cfg.dynamicSmemBytes = smem;
            cfg.stream = st;
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            attr[0].val.programmaticStreamSerializationAllowed = 1;
            cfg.attrs = attr;
            cfg.numAttrs = pdl;
            cudaLaunchKernelEx(&cfg, stream_kernel, s, per_cta, c.S, c.chunk, c.ncons, pdl, sink);
          }
        };
        cudaGraphExec_t ge = nullptr;
        if (graph) {
          cudaGraph_t g;
          cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
          launch_all();
          cudaStreamEndCapture(st, &g);
          cudaGraphInstantiate(&ge, g, 0);
          cudaGraphDestroy(g);
        }
        for (int w = 0; w < 2; ++w) { if (graph) cudaGraphLaunch(ge, st); else launch_all(); }
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0, st);
        for (int w = 0; w < 3; ++w) { if (graph) cudaGraphLaunch(ge, st); else launch_all(); }
        cudaEventRecord(e1, st);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        gbs[mode] = double(per_cta) * sms * reps * 3 / (ms * 1e-3) / 1e9;
        cudaError_t err = cudaGetLastError();
        if (err != cudaSuccess) printf("error %s\n", cudaGetErrorString(err));
        if (ge) cudaGraphExecDestroy(ge);
      }
      printf("%6d %6u %6zu | %8.1f | %8.0f | %8.0f | %8.0f | %8.0f\n", c.S, c.chunk, smem >> 10,
             bytes / 1e6, gbs[0], gbs[1], gbs[2], gbs[3]);
    }
  }
  return 0;
}
