// Calibration microbenchmark (not part of the product): the skeleton of a
// chain of dependent GEMM launches (programmatic dependent launch, CUDA graph),
// with the GEMM work replaced by knobs, to find the per-launch floor.
//
// Per launch: every CTA bulk-copies its share of a weight replica (rotated
// across R replicas, cold in HBM) into shared memory — before
// griddepcontrol.wait when `pre` is set — then waits, reads X (global, 8 KB),
// spins `spin` cycles after its data landed (stand-in for dequant + MMA), and
// writes 64 halves of Y.
//
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/_build/chain_bench tools/chain_bench.cu -lcuda
// run:   tools/_build/chain_bench
#include <cuda_fp16.h>
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

struct P {
  const uint8_t* w;
  uint32_t per_cta;  // bytes per CTA
  int pre, wait, spin, chunks;
  const __half* x;
  __half* y;
  int trig_late;
  int xmode;
};

__global__ void chain_kernel(P p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t base = smem_u32(smem);
  const uint32_t bar = base + p.per_cta;
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    mbar_init(bar + 8, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (!p.trig_late) asm volatile("griddepcontrol.launch_dependents;" :::);
  const uint8_t* src = p.w + static_cast<size_t>(blockIdx.x) * p.per_cta;
  const uint32_t chunk = p.per_cta / p.chunks;
  if (threadIdx.x == 0 && p.per_cta) {
    if (p.pre) {
      mbar_expect(bar, p.per_cta);
      for (int c = 0; c < p.chunks; ++c) bulk(base + c * chunk, src + c * chunk, chunk, bar);
    }
  }
  if (p.wait) asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0 && p.per_cta && !p.pre) {
    mbar_expect(bar, p.per_cta);
    for (int c = 0; c < p.chunks; ++c) bulk(base + c * chunk, src + c * chunk, chunk, bar);
  }
  float acc = 0.f;
  if (p.xmode == 1 && threadIdx.x < 32) {
    for (int i = threadIdx.x; i < 4096; i += 32) acc += __half2float(p.x[i]);
  }
  if (p.xmode == 2) {
    const uint32_t xbar = bar + 8;
    if (threadIdx.x == 0) {
      mbar_expect(xbar, 8192);
      bulk(base + p.per_cta + 64, p.x, 8192, xbar);
    }
    mbar_wait(xbar, 0);
    acc = __half2float(reinterpret_cast<const __half*>(smem + p.per_cta + 64)[threadIdx.x]);
  }
  if (p.per_cta) mbar_wait(bar, 0);
  if (p.trig_late) asm volatile("griddepcontrol.launch_dependents;" :::);
  if (p.spin) {
    long long t0 = clock64();
    while (clock64() - t0 < p.spin) {
    }
  }
  if (threadIdx.x < 64) p.y[blockIdx.x * 64 + threadIdx.x] = __float2half(acc + (p.per_cta ? smem[threadIdx.x] : 0));
}

int main() {
  const int R = 24;
  const size_t per_rep = 8700000;
  uint8_t* w;
  cudaMalloc(&w, R * per_rep + 4096);
  cudaMemset(w, 1, R * per_rep);
  __half *x, *y;
  cudaMalloc(&x, 1 << 20);
  cudaMalloc(&y, 1 << 20);
  cudaMemset(x, 0, 1 << 20);
  cudaFuncSetAttribute(chain_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);

  struct V {
    const char* name;
    int ctas, threads;
    size_t bytes;
    int pre, wait, spin, chunks, pdl, smem_extra, trig_late, xmode;
  };
  std::vector<V> vs = {
      {"truly empty, no PDL", 148, 32, 0, 0, 1, 0, 1, 0, 0, 0, 0},
      {"truly empty, PDL", 148, 32, 0, 0, 1, 0, 1, 1, 0, 0, 0},
      {"truly empty, no wait, PDL", 148, 32, 0, 0, 0, 0, 1, 1, 0, 0, 0},
      {"empty + 1-warp X loop, PDL", 148, 192, 0, 0, 1, 0, 1, 1, 0, 0, 1},
      {"empty, no PDL", 148, 192, 0, 0, 1, 0, 1, 0, 0, 0, 2},
      {"empty, PDL", 148, 192, 0, 0, 1, 0, 1, 1, 0, 0, 2},
      {"empty, PDL, 296 CTAs", 296, 192, 0, 0, 1, 0, 1, 1, 0, 0, 2},
      {"8.7MB prefetch 148, PDL", 148, 192, per_rep, 1, 1, 0, 4, 1, 0, 0, 2},
      {"8.7MB prefetch 296, PDL", 296, 192, per_rep, 1, 1, 0, 4, 1, 0, 0, 2},
      {"8.7MB after-wait 148, PDL", 148, 192, per_rep, 0, 1, 0, 4, 1, 0, 0, 2},
      {"8.7MB prefetch 148, no PDL", 148, 192, per_rep, 1, 1, 0, 4, 0, 0, 0, 2},
      {"8.7MB prefetch 148 +spin 1000", 148, 192, per_rep, 1, 1, 1000, 4, 1, 0, 0, 2},
      {"8.7MB prefetch 148 +spin 2000", 148, 192, per_rep, 1, 1, 2000, 4, 1, 0, 0, 2},
      {"8.7MB prefetch 296 +spin 1000", 296, 192, per_rep, 1, 1, 1000, 4, 1, 0, 0, 2},
      {"8.7MB prefetch 148 +spin 2000, 120KB smem", 148, 192, per_rep, 1, 1, 2000, 4, 1, 120000, 0, 2},
      {"8.7MB prefetch 148 +spin 2000, late trigger", 148, 192, per_rep, 1, 1, 2000, 4, 1, 0, 1, 2},
      {"23MB prefetch 148, PDL", 148, 192, 23000000, 1, 1, 0, 8, 1, 0, 0, 2},
      {"23MB prefetch 296, PDL", 296, 192, 23000000, 1, 1, 0, 8, 1, 0, 0, 2},
  };
  for (const V& v : vs) {
    const uint32_t per_cta = static_cast<uint32_t>(v.bytes / v.ctas) / (16 * v.chunks) * 16 * v.chunks;
    const size_t rep_bytes = v.bytes ? v.bytes : 1;
    const int reps_avail = static_cast<int>((R * per_rep) / rep_bytes);
    const int nrep = reps_avail < 1 ? 1 : reps_avail;
    const size_t smem = per_cta + 64 + 8192 + v.smem_extra;
    auto launch = [&](int i) {
      P p{w + static_cast<size_t>(i % nrep) * rep_bytes, per_cta, v.pre, v.wait, v.spin, v.chunks,
          x, y, v.trig_late, v.xmode};
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(v.ctas);
      cfg.blockDim = dim3(v.threads);
      cfg.dynamicSmemBytes = smem;
      cfg.stream = st;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = at;
      cfg.numAttrs = v.pdl ? 1 : 0;
      cudaLaunchKernelEx(&cfg, chain_kernel, p);
    };
    const int L = 60;
    cudaGraph_t g;
    cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
    for (int i = 0; i < L; ++i) launch(i);
    cudaStreamEndCapture(st, &g);
    cudaGraphExec_t ge;
    cudaGraphInstantiate(&ge, g, 0);
    for (int i = 0; i < 3; ++i) cudaGraphLaunch(ge, st);
    cudaStreamSynchronize(st);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, st);
    for (int i = 0; i < 10; ++i) cudaGraphLaunch(ge, st);
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double us = ms * 1e3 / (10 * L);
    printf("%-46s reps=%2d  %7.3f us/launch  %7.1f GB/s  (%s)\n", v.name, nrep, us,
           v.bytes ? v.bytes / us / 1e3 : 0.0, cudaGetErrorString(cudaGetLastError()));
    cudaGraphExecDestroy(ge);
    cudaGraphDestroy(g);
  }
  return 0;
}
