// flute-b200 — host input producers: NormalFloat tables and the group
// quantizer.  Restates the reference algorithms (nf_table.cpp:18-114,
// quantize.cpp:12-139) with the same floating-point operation order so the
// tables and indices are bit-identical (pinned by tests/test_host_api.py
// against the oracle and the reference library).
#include <algorithm>
#include <cmath>
#include <string>

#include "flutesim/errors.hpp"
#include "flutesim/nf_table.hpp"
#include "flutesim/quantize.hpp"

namespace flutesim {
namespace {

// Acklam's published rational approximation, upper half p in [0.5, 1).
double acklam(double p) {
  constexpr double a0 = -3.969683028665376e+01, a1 = 2.209460984245205e+02,
                   a2 = -2.759285104469687e+02, a3 = 1.383577518672690e+02,
                   a4 = -3.066479806614716e+01, a5 = 2.506628277459239e+00;
  constexpr double b0 = -5.447609879822406e+01, b1 = 1.615858368580409e+02,
                   b2 = -1.556989798598866e+02, b3 = 6.680131188771972e+01,
                   b4 = -1.328068155288572e+01;
  constexpr double c0 = -7.784894002430293e-03, c1 = -3.223964580411365e-01,
                   c2 = -2.400758277161838e+00, c3 = -2.549732539343734e+00,
                   c4 = 4.374664141464968e+00, c5 = 2.938163982698783e+00;
  constexpr double d0 = 7.784695709041462e-03, d1 = 3.224671290700398e-01,
                   d2 = 2.445134137142996e+00, d3 = 3.754408661907416e+00;
  if (p <= 1.0 - 0.02425) {
    const double q = p - 0.5;
    const double r = q * q;
    const double num = (((((a0 * r + a1) * r + a2) * r + a3) * r + a4) * r + a5) * q;
    const double den = ((((b0 * r + b1) * r + b2) * r + b3) * r + b4) * r + 1.0;
    return num / den;
  }
  const double q = std::sqrt(-2.0 * std::log(1.0 - p));
  const double num = ((((c0 * q + c1) * q + c2) * q + c3) * q + c4) * q + c5;
  const double den = (((d0 * q + d1) * q + d2) * q + d3) * q + 1.0;
  return -num / den;
}

double halley_step(double x, double p) {
  const double e = 0.5 * std::erfc(-x / 1.4142135623730951) - p;
  const double u = e * 2.5066282746310002 * std::exp(0.5 * x * x);
  return x - u / (1.0 + 0.5 * x * u);
}

bool is_pow2(int v) { return v > 0 && (v & (v - 1)) == 0; }

// Nearest table value, ties to the smaller index (binary search neighbours).
int nearest_value(const std::vector<float>& v, float r) {
  const auto it = std::lower_bound(v.begin(), v.end(), r);
  if (it == v.begin()) return 0;
  if (it == v.end()) return static_cast<int>(v.size()) - 1;
  const int hi = static_cast<int>(it - v.begin());
  return (v[hi] - r) < (r - v[hi - 1]) ? hi : hi - 1;
}

}  // namespace

double inverse_normal_cdf(double p) {
  if (!(p > 0.0 && p < 1.0)) {
    throw DomainError("inverse_normal_cdf: p must lie in (0,1), got " + std::to_string(p));
  }
  if (p == 0.5) return 0.0;
  if (p < 0.5) return -inverse_normal_cdf(1.0 - p);
  return halley_step(halley_step(acklam(p), p), p);
}

double nf_delta() { return 0.5 * (1.0 / 30.0 + 1.0 / 32.0); }

double nf_sigma() { return 1.0 / inverse_normal_cdf(1.0 - nf_delta()); }

std::vector<double> nf_probability_grid(int bits) {
  if (bits < 2 || bits > 4) {
    throw ConfigError("NormalFloat tables support 2..4 bits, got " + std::to_string(bits));
  }
  const double d = nf_delta();
  const int half = 1 << (bits - 1);
  std::vector<double> p(static_cast<std::size_t>(1) << bits);
  p[0] = d;
  p[half - 1] = 0.5;
  p[p.size() - 1] = 1.0 - d;
  for (int i = 1; i < half - 1; ++i) p[i] = d + (0.5 - d) * i / (half - 1);
  for (int j = 1; j < half; ++j) p[half - 1 + j] = 0.5 + (0.5 - d) * j / half;
  return p;
}

std::vector<double> nf_quantiles(int bits) {
  std::vector<double> q = nf_probability_grid(bits);
  for (double& v : q) v = inverse_normal_cdf(v);
  return q;
}

LookupTable build_nf_table(int bits) {
  const std::vector<double> q = nf_quantiles(bits);
  LookupTable t;
  t.bits = bits;
  t.delta = static_cast<float>(nf_delta());
  for (const double v : q) {
    t.raw_quantiles.push_back(static_cast<float>(v));
    t.values.push_back(static_cast<float>(v / q.back()));
  }
  for (std::size_t i = 1; i < t.values.size(); ++i) {
    if (!(t.values[i - 1] < t.values[i])) {
      throw InternalError("NormalFloat table is not strictly increasing");
    }
  }
  return t;
}

void QuantConfig::validate(int k) const {
  if (bits < 2 || bits > 4) {
    throw ConfigError("quantization bits must be in {2,3,4}, got " + std::to_string(bits));
  }
  if (!is_pow2(group_size) || group_size < 32 || group_size > 256) {
    throw ConfigError("group size must be a power of two in [32, 256], got " +
                      std::to_string(group_size));
  }
  if (k >= 0 && k % group_size != 0) {
    throw ConfigError("quantized dimension " + std::to_string(k) +
                      " is not divisible by group size " + std::to_string(group_size));
  }
}

QuantizedMatrix quantize_matrix(const MatF& w, const QuantConfig& cfg) {
  cfg.validate(w.rows);
  const int k = w.rows, n = w.cols, g = cfg.group_size, gpc = k / g;
  QuantizedMatrix q;
  q.k = k;
  q.n = n;
  q.cfg = cfg;
  q.table = build_nf_table(cfg.bits);
  q.indices.assign(static_cast<std::size_t>(k) * n, 0);
  q.scales.assign(static_cast<std::size_t>(gpc) * n, Half{});

  std::vector<float> absmax(static_cast<std::size_t>(gpc) * n, 0.0f);
  for (int i = 0; i < k; ++i) {
    for (int j = 0; j < n; ++j) {
      const float v = w(i, j);
      if (!std::isfinite(v)) {
        // report the first hit of the reference's j-major scan (quantize.cpp:44-63)
        for (int jj = 0; jj < n; ++jj)
          for (int ii = 0; ii < k; ++ii)
            if (!std::isfinite(w(ii, jj)))
              throw InputError("quantize: non-finite weight at (" + std::to_string(ii) + ", " +
                               std::to_string(jj) + ")");
      }
      float& s = absmax[static_cast<std::size_t>(j) * gpc + i / g];
      s = std::max(s, std::abs(v));
    }
  }
  const long groups = static_cast<long>(gpc) * n;
  for (long gi = 0; gi < groups; ++gi) {
    const Half h = f32_to_f16(absmax[gi]);
    if ((h.bits & 0x7C00u) == 0x7C00u) {
      throw InputError("quantize: group " + std::to_string(gi) + " absmax overflows binary16");
    }
    q.scales[gi] = h;
  }
  const auto zero = static_cast<std::uint8_t>(q.table.zero_index());
#pragma omp parallel for schedule(static)
  for (long gi = 0; gi < groups; ++gi) {
    const int j = static_cast<int>(gi / gpc);
    const int i0 = static_cast<int>(gi % gpc) * g;
    const float s = absmax[gi];
    for (int i = i0; i < i0 + g; ++i) {
      q.indices[static_cast<std::size_t>(i) * n + j] =
          s == 0.0f ? zero : static_cast<std::uint8_t>(nearest_value(q.table.values, w(i, j) / s));
    }
  }
  return q;
}

MatF dequantize_matrix(const QuantizedMatrix& q) {
  MatF out(q.k, q.n);
  for (int i = 0; i < q.k; ++i) {
    for (int j = 0; j < q.n; ++j) {
      out(i, j) = f16_to_f32(q.scales[q.group_of(i, j)]) *
                  q.table.values[q.indices[static_cast<std::size_t>(i) * q.n + j]];
    }
  }
  return out;
}

}  // namespace flutesim
