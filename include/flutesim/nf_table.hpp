// flute-b200 — NormalFloat lookup tables (reference: proj/include/flutesim/
// nf_table.hpp:12-48, algorithm nf_table.cpp:18-114).  Input producer for the
// hot path: the kernel takes T as data (2^b values, narrowed to binary16 by
// make_vectorized_lut), so any table — NF or learned — works.
#pragma once

#include <vector>

namespace flutesim {

struct LookupTable {
  int bits = 0;
  std::vector<float> values;         // normalized, strictly increasing, [-1, 1]
  std::vector<float> raw_quantiles;  // unnormalized Gaussian quantiles
  float delta = 0.0f;

  int index_count() const { return 1 << bits; }
  int zero_index() const { return (1 << (bits - 1)) - 1; }
};

double inverse_normal_cdf(double p);
double nf_delta();
double nf_sigma();
std::vector<double> nf_probability_grid(int bits);
std::vector<double> nf_quantiles(int bits);
LookupTable build_nf_table(int bits);

}  // namespace flutesim
