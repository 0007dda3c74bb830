// flute-b200 — device side of the N-column-sharded layer (host: host_shard.cpp;
// SURVEY.md §8(e)).
//
//  * relayout: NCCL's all-gather of the ranks' [m][w] column slices is
//    shard-major [P][m][w]; Y is row-major [m][n] with rank r's columns at
//    [n0_r, n0_r + w_r).  (m = 1 with equal slices needs no relayout: the
//    all-gather lands straight in Y.)
//  * peer barrier: after the GEMM whose epilogue stored this rank's columns
//    into every rank's Y buffer (peer pointers), thread r publishes
//    "rank `me` finished epoch e of buffer b" into rank r's flag array with a
//    system-scope release store, then waits (acquire) until every rank has
//    published epoch e into this rank's flags — Y buffer b is then complete
//    here.  The release is cumulative over the GEMM kernel's peer stores,
//    which precede it in stream order.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <string>

#include "flutesim/errors.hpp"
#include "ptx.cuh"

namespace flute_dev {

namespace {

__global__ void relayout_kernel(const __half* __restrict__ gathered, __half* __restrict__ y, int m, int n,
                                int world, int w_max, const int* __restrict__ n0s) {
  // one thread per output element of rank r's slice (grid-stride)
  const size_t total = static_cast<size_t>(world) * m * w_max;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const int c = static_cast<int>(i % w_max);
    const size_t rm = i / w_max;
    const int row = static_cast<int>(rm % m);
    const int r = static_cast<int>(rm / m);
    const int col = n0s[r] + c;
    if (col < n0s[r + 1]) y[static_cast<size_t>(row) * n + col] = gathered[i];
  }
}

__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

struct PeerFlags {
  uint32_t* flags[8];  // rank r's flag array [2][world]
};

__global__ void peer_barrier_kernel(PeerFlags pf, int world, int me, int b, uint32_t epoch) {
  const int r = threadIdx.x;
  if (r < world) {
    st_release_sys(pf.flags[r] + b * world + me, epoch);
    const uint32_t* mine = pf.flags[me] + b * world + r;
    while (static_cast<int32_t>(ld_acquire_sys(mine) - epoch) < 0) {
    }
  }
}

[[noreturn]] void fail(const char* what, cudaError_t e) {
  throw flutesim::CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

}  // namespace

void shard_relayout(const void* gathered, void* y, int m, int n, int world, int w_max, const int* n0s_dev,
                    void* stream) {
  const size_t total = static_cast<size_t>(world) * m * w_max;
  const unsigned blocks = static_cast<unsigned>(std::min<size_t>((total + 255) / 256, 148 * 8));
  relayout_kernel<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const __half*>(gathered), static_cast<__half*>(y), m, n, world, w_max, n0s_dev);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) fail("shard relayout", e);
}

void peer_barrier(uint32_t* const* flags, int world, int me, int b, uint32_t epoch, void* stream) {
  if (world < 1 || world > 8) throw flutesim::ConfigError("peer barrier: world must be 1..8");
  PeerFlags pf{};
  for (int r = 0; r < world; ++r) pf.flags[r] = flags[r];
  peer_barrier_kernel<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(pf, world, me, b, epoch);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) fail("peer barrier", e);
}

}  // namespace flute_dev
