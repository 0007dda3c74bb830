// flute-b200 — learned-sigma refinement API (reference: proj/src/quantize.cpp:
// 141-282).  Validation and result assembly follow the reference statement by
// statement; every evaluation runs on the GPU through SteDevice
// (refine_kernels.cu), with W and X uploaded once per call and sigma kept on
// the device between descent steps.
#include <cmath>
#include <string>

#include "device_api.h"
#include "flutesim/errors.hpp"
#include "flutesim/quantize.hpp"

namespace flutesim {

namespace {

void check_inputs(const MatF& w, const MatF& x_calib, const QuantConfig& cfg) {
  cfg.validate(w.rows);  // quantize.cpp:143
  if (x_calib.cols != w.rows) {
    throw InputError("calibration matrix has " + std::to_string(x_calib.cols) +
                     " columns, weights have " + std::to_string(w.rows) + " rows");
  }
}

}  // namespace

SteEval ste_evaluate(const MatF& w, const MatF& x_calib, const QuantConfig& cfg,
                     std::span<const double> sigma_tilde) {
  check_inputs(w, x_calib, cfg);
  const long total_groups = static_cast<long>(w.rows / cfg.group_size) * w.cols;
  if (sigma_tilde.size() != static_cast<std::size_t>(total_groups)) {
    throw InputError("sigma_tilde has wrong group count");
  }
  flute_dev::SteDevice dev(w.data.data(), x_calib.data.data(), x_calib.rows, w.rows, w.cols,
                           cfg.group_size, nf_quantiles(cfg.bits));
  dev.set_sigma(sigma_tilde.data());
  SteEval eval;
  eval.loss = dev.evaluate();
  eval.grad.resize(total_groups);
  eval.indices.resize(static_cast<std::size_t>(w.rows) * w.cols);
  dev.get(nullptr, eval.grad.data(), eval.indices.data(), nullptr);
  return eval;
}

RefineResult refine_scales(const MatF& w, const MatF& x_calib, const QuantConfig& cfg, int steps,
                           double lr) {
  if (steps < 0) throw InputError("refine_scales: steps must be >= 0");
  RefineResult result;
  result.quantized = quantize_matrix(w, cfg);
  check_inputs(w, x_calib, cfg);
  const long total_groups = static_cast<long>(result.quantized.scales.size());
  const double sigma = nf_sigma();
  result.sigma_tilde.assign(total_groups, sigma);

  flute_dev::SteDevice dev(w.data.data(), x_calib.data.data(), x_calib.rows, w.rows, w.cols,
                           cfg.group_size, nf_quantiles(cfg.bits));
  dev.set_sigma(result.sigma_tilde.data());
  if (steps == 0) {
    result.initial_loss = result.final_loss = dev.evaluate();
    return result;
  }
  for (int step = 0; step < steps; ++step) {
    const double loss = dev.evaluate();
    if (!std::isfinite(loss)) throw OptimizationError("refine_scales: loss diverged", step);
    if (step == 0) result.initial_loss = loss;
    dev.descend(lr);
  }
  const double final_loss = dev.evaluate();
  if (!std::isfinite(final_loss)) throw OptimizationError("refine_scales: loss diverged", steps);
  result.final_loss = final_loss;
  std::vector<float> absmax(total_groups);
  dev.get(result.sigma_tilde.data(), nullptr, result.quantized.indices.data(), absmax.data());

  // Fold the learned factor into the stored scale (quantize.cpp:264-280).
  for (long g = 0; g < total_groups; ++g) {
    const double folded = static_cast<double>(absmax[g]) * result.sigma_tilde[g] / sigma;
    if (!(folded >= 0.0) || !std::isfinite(folded)) {
      throw OptimizationError("refine_scales: folded scale is negative or non-finite", steps);
    }
    const Half h = f32_to_f16(static_cast<float>(folded));
    if ((h.bits & 0x7C00u) == 0x7C00u) {
      throw OptimizationError("refine_scales: folded scale overflows binary16", steps);
    }
    result.quantized.scales[g] = h;
  }
  return result;
}

}  // namespace flutesim
