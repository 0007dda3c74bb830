// Calibration microbenchmark (not part of the product): per-launch time of a
// CUDA graph of back-to-back launches that do no work, to separate the
// launch / programmatic-dependent-launch floor from the GEMM kernel's own
// prologue and epilogue.  Variants: plain / PDL, grid 148 / 256 / 296, with
// ~110 KB dynamic shared memory (two CTAs per SM, as the LUT-GEMM), with
// thread-block clusters of 4, with an mbarrier init + CTA barrier prologue.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/_build/launch_floor tools/launch_floor.cu
#include <cuda_runtime.h>
#include <cstdio>

__global__ void empty_kernel(int mode, unsigned* sink) {
  extern __shared__ __align__(16) unsigned char smem[];
  if (mode & 1) {  // prologue: mbarrier init + fence + __syncthreads
    if (threadIdx.x == 0) {
      unsigned bar = static_cast<unsigned>(__cvta_generic_to_shared(smem));
      for (int i = 0; i < 16; ++i)
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar + 8 * i), "r"(1) : "memory");
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
  }
  if (mode & 2) {  // cluster barrier (arrive + wait), as the cluster split-K prologue
    asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
    asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
  }
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (mode & 4) {  // a global store per CTA after the wait (as Y)
    if (threadIdx.x == 0) sink[blockIdx.x] = blockIdx.x;
  }
}

int main() {
  unsigned* sink;
  cudaMalloc(&sink, 4096 * 4);
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  const int smem = 110 * 1024;
  cudaFuncSetAttribute(empty_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  struct V { int grid, pdl, cluster, mode, sm; const char* name; };
  V vs[] = {{148, 0, 1, 0, 0, "148 CTAs, no PDL, no smem"}, {148, 1, 1, 0, 0, "148 CTAs, PDL, no smem"},
            {256, 1, 1, 0, smem, "256 CTAs, PDL, 110 KB"}, {296, 1, 1, 0, smem, "296 CTAs, PDL, 110 KB"},
            {256, 1, 4, 0, smem, "256 CTAs, PDL, 110 KB, cluster 4"},
            {256, 1, 4, 2, smem, "  + cluster barrier"}, {256, 1, 4, 3, smem, "  + mbarrier init"},
            {256, 1, 4, 7, smem, "  + Y store"}, {224, 1, 1, 5, smem, "224 CTAs, PDL, 110 KB, init + store"},
            {224, 0, 1, 5, smem, "224 CTAs, no PDL, 110 KB, init + store"}};
  for (const V& v : vs) {
    const int L = 20;
    auto launch_all = [&]() {
      for (int i = 0; i < L; ++i) {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(v.grid);
        cfg.blockDim = dim3(192);
        cfg.dynamicSmemBytes = v.sm;
        cfg.stream = st;
        cudaLaunchAttribute attr[2];
        int na = 0;
        if (v.pdl) {
          attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
          attr[na].val.programmaticStreamSerializationAllowed = 1;
          ++na;
        }
        if (v.cluster > 1) {
          attr[na].id = cudaLaunchAttributeClusterDimension;
          attr[na].val.clusterDim.x = v.cluster;
          attr[na].val.clusterDim.y = 1;
          attr[na].val.clusterDim.z = 1;
          ++na;
        }
        cfg.attrs = attr;
        cfg.numAttrs = na;
        cudaLaunchKernelEx(&cfg, empty_kernel, v.mode, sink);
      }
    };
    cudaGraph_t g;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
    launch_all();
    cudaStreamEndCapture(st, &g);
    cudaGraphInstantiate(&ge, g, 0);
    for (int w = 0; w < 3; ++w) cudaGraphLaunch(ge, st);
    cudaStreamSynchronize(st);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, st);
    for (int r = 0; r < 10; ++r) cudaGraphLaunch(ge, st);
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("%-45s %6.2f us per launch  (%s)\n", v.name, ms * 1e3 / (10 * L), cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
