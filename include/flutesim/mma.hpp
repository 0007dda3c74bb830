// flute-b200 — fragment MMA (reference: proj/include/flutesim/mma.hpp:15-24,
// mma.cpp:10-30).
//
// In the reference this is a scalar simulation of a 16x8x16 tensor-core MMA.
// Here mma_fragment runs on the B200 tensor cores: the fragments are uploaded
// and issued as mma.sync.m16n8k16.f32.f16.f16.f32 tiles (SASS HMMA.16816.F32),
// fp32 accumulate.  The reference's contract — error within
// k * 2^-24 * max|a row| * max|b col| of binary64, bitwise deterministic — holds;
// the per-k summation order inside the tensor core is the hardware's.
#pragma once

#include <span>

#include "flutesim/half.hpp"

namespace flutesim {

struct FragDims {
  int m = 16;
  int n = 8;
  int k = 16;
};

// c[m][n] += sum_k a[m][k] * b[k][n]; all row-major.  Any positive dims: the
// operands are zero-padded on the device to whole 16x8x16 atoms (padding adds
// exact zeros).  ConfigError on non-positive dims or span-size mismatch.
void mma_fragment(std::span<const Half> a, std::span<const Half> b, std::span<float> c,
                  const FragDims& dims);

}  // namespace flutesim
