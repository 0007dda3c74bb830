// flute-b200 — learned-sigma scale refinement on the GPU (
// reference: proj/src/quantize.cpp:141-282, ste_evaluate / refine_scales).
//
// One straight-through evaluation of L = ||X (W_hat - W)||_F^2 is four passes
// over device-resident W (f32 [k][n]) and X (f32 [m][k]):
//   1. requant_kernel   per (group, column): absmax, candidates absmax*sigma*q_c,
//                       nearest index (ties to the lower index), D = W_hat - W
//                       (quantize.cpp:167-190);
//   2. gemm_f64_kernel  E = X D          ([m][n], quantize.cpp:192-205);
//   3. sumsq_kernel     loss = sum E^2   (:206-208);
//   4. gemm_f64_kernel  G = X^T E        ([k][n]), then
//      grad_kernel      grad_g = sum_{i in g} ((2 G_ij) absmax_g) q_c(i,j) (:210-228).
// Every product and sum is an explicit binary64 __dmul_rn / __dadd_rn in the
// reference's order (p ascending inside each dot product, i ascending inside
// each group), so indices, E, G and the gradients are bit-identical to the
// reference's scalar loops (no FMA contraction on either side).  The loss is a
// fixed-order tree sum (deterministic; equal to the reference's sequential sum
// to ~1e-15 relative).  The descent update sigma -= lr * grad runs on the
// device too, so refine_scales moves only the loss (8 bytes) per step.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <string>
#include <vector>

#include "device_api.h"
#include "flutesim/errors.hpp"

namespace flute_dev {
namespace refine {

constexpr unsigned long long kNoBad = ~0ull;

// thread = (group row G, column j), consecutive threads = consecutive columns
__global__ void requant_kernel(const float* __restrict__ w, int k, int n, int group, int nq,
                               const double* __restrict__ q, const double* __restrict__ sigma,
                               std::uint8_t* __restrict__ idx, double* __restrict__ d,
                               float* __restrict__ absmax, unsigned long long* __restrict__ bad) {
  const int gpc = k / group;
  const long tid = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (tid >= static_cast<long>(gpc) * n) return;
  const int j = static_cast<int>(tid % n);
  const int G = static_cast<int>(tid / n);
  const long g = static_cast<long>(j) * gpc + G;
  const int i0 = G * group;
  float amax = 0.f;
  for (int i = i0; i < i0 + group; ++i) {
    const float v = w[static_cast<size_t>(i) * n + j];
    if (!isfinite(v)) {
      // the reference scans j-major (quantize.cpp:44-63): report its first hit
      atomicMin(bad, static_cast<unsigned long long>(j) * k + i);
      return;
    }
    const float a = fabsf(v);
    amax = amax < a ? a : amax;  // std::max(s, |v|)
  }
  absmax[g] = amax;
  if (amax == 0.0f) {
    const auto zero = static_cast<std::uint8_t>((1 << (nq == 16 ? 3 : nq == 8 ? 2 : 1)) - 1);
    for (int i = i0; i < i0 + group; ++i) {
      const size_t e = static_cast<size_t>(i) * n + j;
      idx[e] = zero;
      d[e] = __dsub_rn(0.0, static_cast<double>(w[e]));
    }
    return;
  }
  const double eff = __dmul_rn(static_cast<double>(amax), sigma[g]);
  double cand[16];
#pragma unroll
  for (int c = 0; c < 16; ++c)
    if (c < nq) cand[c] = __dmul_rn(eff, q[c]);
  for (int i = i0; i < i0 + group; ++i) {
    const size_t e = static_cast<size_t>(i) * n + j;
    const double u = static_cast<double>(w[e]);
    int best = 0;
    double bd = fabs(__dsub_rn(cand[0], u));
#pragma unroll
    for (int c = 1; c < 16; ++c) {
      if (c < nq) {
        const double dc = fabs(__dsub_rn(cand[c], u));
        if (dc < bd) {
          bd = dc;
          best = c;
        }
      }
    }
    idx[e] = static_cast<std::uint8_t>(best);
    double wh = cand[0];
#pragma unroll
    for (int c = 1; c < 16; ++c)
      if (c == best) wh = cand[c];
    d[e] = __dsub_rn(wh, u);
  }
}

// C[R][N] = sum_p A(r, p) * B[p][c], A f32 at a[r*sar + p*sap] (widened
// exactly), B f64 row-major [P][N].  64x64 output tile per CTA, 16-deep p
// slabs through shared memory, 4x4 outputs per thread, p ascending.
constexpr int kTR = 64, kTC = 64, kTP = 16;
__global__ void __launch_bounds__(256) gemm_f64_kernel(const float* __restrict__ a, long sar,
                                                       long sap, const double* __restrict__ b,
                                                       double* __restrict__ c, int R, int N,
                                                       int P) {
  __shared__ double As[kTP][kTR + 1];
  __shared__ double Bs[kTP][kTC];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const int r0 = blockIdx.y * kTR, c0 = blockIdx.x * kTC;
  double acc[4][4];
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) acc[u][v] = 0.0;
  for (int p0 = 0; p0 < P; p0 += kTP) {
    const int pn = P - p0 < kTP ? P - p0 : kTP;
    // A slab: 64 rows x 16 p; lanes walk whichever index is contiguous in memory
    for (int e = threadIdx.x; e < kTR * kTP; e += 256) {
      int rr, pp;
      if (sap == 1) {
        rr = e / kTP;
        pp = e % kTP;
      } else {
        rr = e % kTR;
        pp = e / kTR;
      }
      const int r = r0 + rr, p = p0 + pp;
      As[pp][rr] = (r < R && pp < pn) ? static_cast<double>(a[r * sar + p * sap]) : 0.0;
    }
    for (int e = threadIdx.x; e < kTP * kTC; e += 256) {
      const int pp = e / kTC, cc = e % kTC;
      const int cg = c0 + cc, p = p0 + pp;
      Bs[pp][cc] = (cg < N && pp < pn) ? b[static_cast<size_t>(p) * N + cg] : 0.0;
    }
    __syncthreads();
    for (int pp = 0; pp < pn; ++pp) {
      double av[4], bv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) av[u] = As[pp][ty * 4 + u];
#pragma unroll
      for (int v = 0; v < 4; ++v) bv[v] = Bs[pp][tx + 16 * v];
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[u][v] = __dadd_rn(acc[u][v], __dmul_rn(av[u], bv[v]));
    }
    __syncthreads();
  }
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int r = r0 + ty * 4 + u;
    if (r >= R) continue;
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int cg = c0 + tx + 16 * v;
      if (cg < N) c[static_cast<size_t>(r) * N + cg] = acc[u][v];
    }
  }
}

// loss = sum e^2: one CTA, fixed per-thread strides then a fixed tree.
__global__ void __launch_bounds__(1024) sumsq_kernel(const double* __restrict__ e, long count,
                                                     double* __restrict__ out) {
  __shared__ double part[1024];
  double s = 0.0;
  for (long i = threadIdx.x; i < count; i += 1024) s = __dadd_rn(s, __dmul_rn(e[i], e[i]));
  part[threadIdx.x] = s;
  __syncthreads();
  for (int h = 512; h > 0; h >>= 1) {
    if (threadIdx.x < h) part[threadIdx.x] = __dadd_rn(part[threadIdx.x], part[threadIdx.x + h]);
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = part[0];
}

__global__ void grad_kernel(const double* __restrict__ gm, const std::uint8_t* __restrict__ idx,
                            const float* __restrict__ absmax, const double* __restrict__ q, int k,
                            int n, int group, double* __restrict__ grad) {
  const int gpc = k / group;
  const long tid = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (tid >= static_cast<long>(gpc) * n) return;
  const int j = static_cast<int>(tid % n);
  const int G = static_cast<int>(tid / n);
  const long g = static_cast<long>(j) * gpc + G;
  const double am = static_cast<double>(absmax[g]);
  double acc = 0.0;
  if (absmax[g] != 0.0f) {
    for (int i = G * group; i < (G + 1) * group; ++i) {
      const size_t e = static_cast<size_t>(i) * n + j;
      acc = __dadd_rn(acc, __dmul_rn(__dmul_rn(__dmul_rn(2.0, gm[e]), am), q[idx[e]]));
    }
  }
  grad[g] = acc;
}

__global__ void descend_kernel(double* __restrict__ sigma, const double* __restrict__ grad,
                               double lr, long groups) {
  const long g = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (g < groups) sigma[g] = __dsub_rn(sigma[g], __dmul_rn(lr, grad[g]));
}

}  // namespace refine

namespace {
void rcheck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw flutesim::CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}
template <class T>
T* rmalloc(size_t count) {
  void* p = nullptr;
  if (count == 0) count = 1;
  rcheck(cudaMalloc(&p, count * sizeof(T)), "cudaMalloc");
  return static_cast<T*>(p);
}
unsigned blocks(long items, int per) { return static_cast<unsigned>((items + per - 1) / per); }
}  // namespace

SteDevice::SteDevice(const float* w, const float* x, int m, int k, int n, int group,
                     const std::vector<double>& quantiles)
    : m_(m), k_(k), n_(n), group_(group), nq_(static_cast<int>(quantiles.size())) {
  int dev_count = 0;
  if (cudaGetDeviceCount(&dev_count) != cudaSuccess || dev_count == 0)
    throw flutesim::CudaError("refine: no CUDA device");
  groups_ = static_cast<long>(k / group) * n;
  const size_t kn = static_cast<size_t>(k) * n;
  w_ = rmalloc<float>(kn);
  x_ = rmalloc<float>(static_cast<size_t>(m) * k);
  q_ = rmalloc<double>(16);
  sigma_ = rmalloc<double>(groups_);
  grad_ = rmalloc<double>(groups_);
  absmax_ = rmalloc<float>(groups_);
  idx_ = rmalloc<std::uint8_t>(kn);
  d_ = rmalloc<double>(kn);  // D, then reused for G = X^T E
  e_ = rmalloc<double>(static_cast<size_t>(m) * n);
  scalars_ = rmalloc<double>(1);
  bad_ = rmalloc<unsigned long long>(1);
  rcheck(cudaMemcpy(w_, w, kn * sizeof(float), cudaMemcpyHostToDevice), "cudaMemcpy");
  rcheck(cudaMemcpy(x_, x, static_cast<size_t>(m) * k * sizeof(float), cudaMemcpyHostToDevice),
         "cudaMemcpy");
  rcheck(cudaMemcpy(q_, quantiles.data(), quantiles.size() * sizeof(double), cudaMemcpyHostToDevice),
         "cudaMemcpy");
}

SteDevice::~SteDevice() {
  for (void* p : {static_cast<void*>(w_), static_cast<void*>(x_), static_cast<void*>(q_),
                  static_cast<void*>(sigma_), static_cast<void*>(grad_), static_cast<void*>(absmax_),
                  static_cast<void*>(idx_), static_cast<void*>(d_), static_cast<void*>(e_),
                  static_cast<void*>(scalars_), static_cast<void*>(bad_)})
    cudaFree(p);
}

void SteDevice::set_sigma(const double* sigma_host) {
  rcheck(cudaMemcpy(sigma_, sigma_host, groups_ * sizeof(double), cudaMemcpyHostToDevice),
         "cudaMemcpy");
}

double SteDevice::evaluate() {
  using namespace refine;
  rcheck(cudaMemset(bad_, 0xFF, sizeof(unsigned long long)), "cudaMemset");
  requant_kernel<<<blocks(groups_, 256), 256>>>(w_, k_, n_, group_, nq_, q_, sigma_, idx_, d_,
                                                absmax_, bad_);
  rcheck(cudaGetLastError(), "requant_kernel");
  unsigned long long bad = kNoBad;
  rcheck(cudaMemcpy(&bad, bad_, sizeof(bad), cudaMemcpyDeviceToHost), "cudaMemcpy");
  if (bad != kNoBad) {
    const long long j = static_cast<long long>(bad / k_), i = static_cast<long long>(bad % k_);
    throw flutesim::InputError("quantize: non-finite weight at (" + std::to_string(i) + ", " +
                               std::to_string(j) + ")");
  }
  // E = X D: rows t (m), cols j (n), p = i (k)
  gemm_f64_kernel<<<dim3(blocks(n_, kTC), blocks(m_, kTR)), 256>>>(x_, k_, 1, d_, e_, m_, n_, k_);
  rcheck(cudaGetLastError(), "gemm_f64_kernel");
  sumsq_kernel<<<1, 1024>>>(e_, static_cast<long>(m_) * n_, scalars_);
  rcheck(cudaGetLastError(), "sumsq_kernel");
  // G = X^T E: rows i (k), cols j (n), p = t (m); overwrites D
  gemm_f64_kernel<<<dim3(blocks(n_, kTC), blocks(k_, kTR)), 256>>>(x_, 1, k_, e_, d_, k_, n_, m_);
  rcheck(cudaGetLastError(), "gemm_f64_kernel");
  grad_kernel<<<blocks(groups_, 256), 256>>>(d_, idx_, absmax_, q_, k_, n_, group_, grad_);
  rcheck(cudaGetLastError(), "grad_kernel");
  double loss = 0.0;
  rcheck(cudaMemcpy(&loss, scalars_, sizeof(double), cudaMemcpyDeviceToHost), "cudaMemcpy");
  return loss;
}

void SteDevice::descend(double lr) {
  refine::descend_kernel<<<blocks(groups_, 256), 256>>>(sigma_, grad_, lr, groups_);
  rcheck(cudaGetLastError(), "descend_kernel");
}

void SteDevice::get(double* sigma, double* grad, std::uint8_t* idx, float* absmax) const {
  if (sigma) rcheck(cudaMemcpy(sigma, sigma_, groups_ * sizeof(double), cudaMemcpyDeviceToHost), "cudaMemcpy");
  if (grad) rcheck(cudaMemcpy(grad, grad_, groups_ * sizeof(double), cudaMemcpyDeviceToHost), "cudaMemcpy");
  if (idx)
    rcheck(cudaMemcpy(idx, idx_, static_cast<size_t>(k_) * n_, cudaMemcpyDeviceToHost), "cudaMemcpy");
  if (absmax)
    rcheck(cudaMemcpy(absmax, absmax_, groups_ * sizeof(float), cudaMemcpyDeviceToHost), "cudaMemcpy");
}

}  // namespace flute_dev
