// flute-b200 — weight-preparation kernels, sm_100a:
//   * quantize_kernel: the group quantizer of quantize.cpp:81-128 on the GPU —
//     per-(column, group) absmax, binary16 scale (RNE), index = nearest table
//     value of w / absmax (IEEE division, ties to the lower index, zero groups
//     to the table's zero index), bit-exact with the reference;
//   * unpack_canonical_kernel: canonical reorder_and_split slices -> indices
//     (packed_pos, pack.cpp:48-63), so an FLTE file can be uploaded as stored
//     and re-permuted on the device;
//   * pack_device_kernel / scales_device_kernel: indices [k][n] and scales
//     [n][k/g] -> the sm_100a device layout (host_pack.cpp is the normative
//     description; tests compare against it byte for byte).
// All are one-thread-per-element gather/scatter passes (offline, HBM-bound).
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <string>

#include "dequant.cuh"
#include "device_api.h"
#include "flutesim/errors.hpp"

namespace flute_dev {
namespace prep {

constexpr int kUnitN = 64, kUnitK = 128;

struct Layout6 {
  int tm, tn, tk, fm, fn, fk;
};

// flags[0] |= 1: non-finite weight; flags[0] |= 2: absmax overflows binary16
__global__ void quantize_kernel(const float* __restrict__ w, int k, int n, int group, int bits,
                                const float* __restrict__ table, uint8_t* __restrict__ idx,
                                uint16_t* __restrict__ scales, unsigned* __restrict__ flags) {
  const int gpc = k / group;
  const long tid = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (tid >= static_cast<long>(gpc) * n) return;
  // consecutive threads = consecutive columns of one group row: coalesced loads
  const int j = static_cast<int>(tid % n);
  const int G = static_cast<int>(tid / n);
  const int i0 = G * group;
  float amax = 0.f;
  bool bad = false;
  for (int i = i0; i < i0 + group; ++i) {
    const float v = w[static_cast<size_t>(i) * n + j];
    bad |= !isfinite(v);
    amax = fmaxf(amax, fabsf(v));
  }
  if (bad) {
    atomicOr(flags, 1u);
    return;
  }
  const __half s16 = __float2half_rn(amax);
  const uint16_t sb = __half_as_ushort(s16);
  if ((sb & 0x7C00u) == 0x7C00u) atomicOr(flags, 2u);
  scales[static_cast<size_t>(j) * gpc + G] = sb;
  const int nv = 1 << bits;
  const uint8_t zero = static_cast<uint8_t>((1 << (bits - 1)) - 1);
  for (int i = i0; i < i0 + group; ++i) {
    uint8_t q = zero;
    if (amax != 0.f) {
      const float r = __fdiv_rn(w[static_cast<size_t>(i) * n + j], amax);
      // lower_bound: first value not less than r
      int hi = 0;
      while (hi < nv && table[hi] < r) ++hi;
      if (hi == 0) {
        q = 0;
      } else if (hi == nv) {
        q = static_cast<uint8_t>(nv - 1);
      } else {
        const float d_lo = __fsub_rn(r, table[hi - 1]);
        const float d_hi = __fsub_rn(table[hi], r);
        q = static_cast<uint8_t>(d_hi < d_lo ? hi : hi - 1);
      }
    }
    idx[static_cast<size_t>(i) * n + j] = q;
  }
}

__device__ __forceinline__ size_t packed_pos(const Layout6& L, int k, int i, int j) {
  const long tiles_k = k / L.tk;
  const long tile = static_cast<long>(j / L.tn) * tiles_k + i / L.tk;
  const int ki = i % L.tk, nj = j % L.tn;
  const long frag = static_cast<long>(ki / L.fk) * (L.tn / L.fn) + nj / L.fn;
  const long within = static_cast<long>(ki % L.fk) * L.fn + nj % L.fn;
  return static_cast<size_t>(tile * static_cast<long>(L.tk) * L.tn + frag * L.fk * L.fn + within);
}

__global__ void unpack_canonical_kernel(const uint32_t* __restrict__ s0, const uint32_t* __restrict__ s1,
                                        int k, int n, int bits, Layout6 L, uint8_t* __restrict__ idx) {
  const long t = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= static_cast<long>(k) * n) return;
  const int i = static_cast<int>(t / n), j = static_cast<int>(t % n);
  const size_t pos = packed_pos(L, k, i, j);
  uint32_t v;
  if (bits == 3) {
    const size_t b2 = pos * 2, b1 = pos;
    const uint32_t hi = (s0[b2 >> 5] >> (b2 & 31)) & 3u;
    const uint32_t lo = (s1[b1 >> 5] >> (b1 & 31)) & 1u;
    v = (hi << 1) | lo;
  } else {
    const size_t b = pos * bits;
    v = (s0[b >> 5] >> (b & 31)) & ((1u << bits) - 1u);
  }
  idx[t] = static_cast<uint8_t>(v);
}

// One thread per (unit, k-step, lane) slot of the device layout.
__global__ void pack_device_kernel(const uint8_t* __restrict__ idx, int k, int n, int bits,
                                   int tiles_k, long units, uint8_t* __restrict__ out) {
  const long t = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= units * 256) return;
  const long u = t >> 8;
  const int slot = static_cast<int>(t & 255);
  const int w = slot >> 5, lane = slot & 31;
  const int nt = static_cast<int>(u / tiles_k), kt = static_cast<int>(u % tiles_k);
  const int gr = lane >> 2, tq = lane & 3;
  const uint32_t zero = (1u << (bits - 1)) - 1u;
  auto at = [&](int row, int col) -> uint32_t {
    return (row < k && col < n) ? idx[static_cast<size_t>(row) * n + col] : zero;
  };
  const size_t ub = static_cast<size_t>(kUnitN) * kUnitK * bits / 8;
  uint8_t* unit = out + static_cast<size_t>(u) * ub;
  uint8_t bytes[16] = {};
  uint32_t d3[16];  // 3-bit: six-bit device indices, encoded by pack_lane_w3
#pragma unroll
  for (int j = 0; j < 4; ++j)
#pragma unroll
    for (int p = 0; p < 4; ++p) {
      const int col = nt * kUnitN + 16 * j + gr + 8 * (p & 1);
      const int row = kt * kUnitK + 16 * w + 2 * tq + 8 * (p >> 1);
      const uint32_t a = at(row, col), b = at(row + 1, col);
      if (bits == 4) {
        bytes[j * 4 + p] = static_cast<uint8_t>((a << 4) | b);
      } else if (bits == 2) {
        bytes[(j >> 1) * 4 + p] |= static_cast<uint8_t>(((a << 2) | b) << (4 * (j & 1)));
      } else {
        d3[4 * j + p] = ((((a >> 1) << 2) | (b >> 1)) << 2) | ((a & 1u) << 1) | (b & 1u);
      }
    }
  if (bits == 4) {
    uint4* d = reinterpret_cast<uint4*>(unit + slot * 16);
    *d = *reinterpret_cast<const uint4*>(bytes);
  } else if (bits == 2) {
    uint2* d = reinterpret_cast<uint2*>(unit + slot * 8);
    *d = *reinterpret_cast<const uint2*>(bytes);
  } else {
    uint32_t wa, wb, wc;
    pack_lane_w3(d3, wa, wb, wc);
    *reinterpret_cast<uint2*>(unit + slot * 8) = make_uint2(wa, wb);
    *reinterpret_cast<uint32_t*>(unit + 2048 + slot * 4) = wc;
  }
}

__global__ void scales_device_kernel(const uint16_t* __restrict__ sc, int k, int n, int group,
                                     int tiles_n, int gp, uint16_t* __restrict__ out) {
  const long t = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= static_cast<long>(tiles_n) * gp * kUnitN) return;
  const int e = static_cast<int>(t % kUnitN);
  const long blk = t / kUnitN;
  const int G = static_cast<int>(blk % gp), nt = static_cast<int>(blk / gp);
  const int gr = e >> 3, j = (e >> 1) & 3, h = e & 1;
  const int col = nt * kUnitN + 16 * j + gr + 8 * h;
  const int gpc = k / group;
  out[t] = (col < n && G < gpc) ? sc[static_cast<size_t>(col) * gpc + G] : 0;
}

}  // namespace prep

namespace {
void prep_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw flutesim::CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}
unsigned grid_for(long items, int block) {
  return static_cast<unsigned>((items + block - 1) / block);
}
}  // namespace

void quantize_device(const float* w, int k, int n, int bits, int group, const float* table_host,
                     uint8_t* idx, uint16_t* scales, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  float* table = nullptr;
  unsigned* flags = nullptr;
  prep_check(cudaMallocAsync(&table, 16 * sizeof(float), st), "cudaMallocAsync");
  prep_check(cudaMallocAsync(&flags, sizeof(unsigned), st), "cudaMallocAsync");
  prep_check(cudaMemcpyAsync(table, table_host, sizeof(float) << bits, cudaMemcpyHostToDevice, st),
             "cudaMemcpyAsync");
  prep_check(cudaMemsetAsync(flags, 0, sizeof(unsigned), st), "cudaMemsetAsync");
  const long items = static_cast<long>(k / group) * n;
  prep::quantize_kernel<<<grid_for(items, 256), 256, 0, st>>>(w, k, n, group, bits, table, idx,
                                                              scales, flags);
  prep_check(cudaGetLastError(), "quantize_kernel");
  unsigned hflags = 0;
  prep_check(cudaMemcpyAsync(&hflags, flags, sizeof(unsigned), cudaMemcpyDeviceToHost, st),
             "cudaMemcpyAsync");
  prep_check(cudaFreeAsync(table, st), "cudaFreeAsync");
  prep_check(cudaFreeAsync(flags, st), "cudaFreeAsync");
  prep_check(cudaStreamSynchronize(st), "cudaStreamSynchronize");
  if (hflags & 1u) throw flutesim::InputError("quantize: non-finite weight");
  if (hflags & 2u) throw flutesim::InputError("quantize: group absmax overflows binary16");
}

void unpack_canonical_device(const uint32_t* s0, const uint32_t* s1, int k, int n, int bits,
                             const int* layout6, uint8_t* idx, void* stream) {
  const prep::Layout6 L{layout6[0], layout6[1], layout6[2], layout6[3], layout6[4], layout6[5]};
  const long items = static_cast<long>(k) * n;
  prep::unpack_canonical_kernel<<<grid_for(items, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      s0, s1, k, n, bits, L, idx);
  prep_check(cudaGetLastError(), "unpack_canonical_kernel");
}

void pack_device_on_device(const uint8_t* idx, int k, int n, int bits, int group, uint8_t* out,
                           void* stream) {
  (void)group;
  const int tiles_k = (k + 127) / 128, tiles_n = (n + 63) / 64;
  const long units = static_cast<long>(tiles_k) * tiles_n;
  prep::pack_device_kernel<<<grid_for(units * 256, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      idx, k, n, bits, tiles_k, units, out);
  prep_check(cudaGetLastError(), "pack_device_kernel");
}

void scales_device_on_device(const uint16_t* sc, int k, int n, int group, uint16_t* out,
                             void* stream) {
  const int tiles_n = (n + 63) / 64;
  const int kp = (k + 127) / 128 * 128;
  const int gp = kp / group;
  const long items = static_cast<long>(tiles_n) * gp * 64;
  prep::scales_device_kernel<<<grid_for(items, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      sc, k, n, group, tiles_n, gp, out);
  prep_check(cudaGetLastError(), "scales_device_kernel");
}

}  // namespace flute_dev
