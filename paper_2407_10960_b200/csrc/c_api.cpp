// flute-b200 — C ABI implementation (include/flute_c.h).  Thin: every entry
// point converts plain pointers to the C++ API and maps exceptions to status
// codes, keeping the message for flute_last_error().
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <exception>
#include <string>

#include "device_api.h"
#include "flute_c.h"
#include "flutesim/engine.hpp"
#include "flutesim/flte.hpp"
#include "flutesim/errors.hpp"
#include "flutesim/mma.hpp"
#include "flutesim/quantize.hpp"
#include "flutesim/sharded.hpp"

using namespace flutesim;

namespace {

thread_local std::string g_last_error;

template <class F>
int guard(F&& f) {
  try {
    f();
    g_last_error.clear();
    return FLUTE_OK;
  } catch (const CudaError& e) {
    g_last_error = e.what();
    return FLUTE_ERR_CUDA;
  } catch (const ConfigError& e) {
    g_last_error = e.what();
    return FLUTE_ERR_CONFIG;
  } catch (const InputError& e) {
    g_last_error = e.what();
    return FLUTE_ERR_INPUT;
  } catch (const InternalError& e) {
    g_last_error = e.what();
    return FLUTE_ERR_INTERNAL;
  } catch (const OptimizationError& e) {
    g_last_error = e.what();
    return FLUTE_ERR_OPTIMIZATION;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return FLUTE_ERR_INTERNAL;
  }
}

LayoutDescriptor to_layout(const int* l) {
  if (l == nullptr) return LayoutDescriptor{};
  return LayoutDescriptor{l[0], l[1], l[2], l[3], l[4], l[5]};
}

void need(const void* p, const char* what) {
  if (p == nullptr) throw InputError(std::string(what) + " is null");
}

PackedWeights canonical_from(const uint32_t* hi, const uint32_t* lo, int k, int n, int bits,
                             const LayoutDescriptor& L) {
  need(hi, "slice_hi");
  if (bits == 3) need(lo, "slice_lo");
  if (k < 1 || n < 1) throw ConfigError("k and n must be positive");
  PackedWeights pw;
  pw.layout = L;
  pw.bits = bits;
  pw.k = k;
  pw.n = n;
  const std::size_t total = static_cast<std::size_t>(k) * n;
  if (bits == 3) {
    pw.slices = {BitSlice{2, std::vector<uint32_t>(hi, hi + (total * 2 + 31) / 32)},
                 BitSlice{1, std::vector<uint32_t>(lo, lo + (total + 31) / 32)}};
  } else {
    pw.slices = {BitSlice{bits, std::vector<uint32_t>(hi, hi + (total * bits + 31) / 32)}};
  }
  return pw;
}

VectorizedTable table_from_words(const uint32_t* words, int bits) {
  need(words, "vlut_words");
  if (bits < 2 || bits > 4) throw ConfigError("bits must be in {2,3,4}");
  VectorizedTable vt;
  vt.bits = bits;
  vt.dup = 1;
  vt.entries.resize(std::size_t{1} << (2 * bits));
  for (std::size_t e = 0; e < vt.entries.size(); ++e) {
    vt.entries[e] = {Half::from_bits(static_cast<uint16_t>(words[e] & 0xFFFFu)),
                     Half::from_bits(static_cast<uint16_t>(words[e] >> 16))};
  }
  return vt;
}

}  // namespace

struct flute_comm {
  std::unique_ptr<Communicator> impl;
};
struct flute_sharded {
  std::unique_ptr<ShardedWeights> impl;
};

struct flute_weights {
  DeviceWeights* impl = nullptr;
  int k = 0, n = 0, bits = 0, group = 0;
};

extern "C" {

const char* flute_last_error(void) { return g_last_error.c_str(); }
const char* flute_version(void) { return "flute-b200 0.1 (sm_100a)"; }

uint16_t flute_f32_to_f16(float x) { return f32_to_f16(x).bits; }
float flute_f16_to_f32(uint16_t h) { return f16_to_f32(Half::from_bits(h)); }

int flute_nf_table(int bits, float* values_out) {
  return guard([&] {
    need(values_out, "values_out");
    const LookupTable t = build_nf_table(bits);
    std::memcpy(values_out, t.values.data(), t.values.size() * sizeof(float));
  });
}

int flute_nf_quantiles(int bits, double* values_out) {
  return guard([&] {
    need(values_out, "values_out");
    const std::vector<double> q = nf_quantiles(bits);
    std::memcpy(values_out, q.data(), q.size() * sizeof(double));
  });
}

double flute_nf_sigma(void) { return nf_sigma(); }

int flute_quantize(const float* w, int k, int n, int bits, int group, uint8_t* indices_out,
                   uint16_t* scales_out) {
  return guard([&] {
    need(w, "w");
    need(indices_out, "indices_out");
    need(scales_out, "scales_out");
    if (k < 1 || n < 1) throw ConfigError("k and n must be positive");
    MatF m(k, n);
    std::memcpy(m.data.data(), w, sizeof(float) * m.data.size());
    const QuantizedMatrix q = quantize_matrix(m, QuantConfig{bits, group});
    std::memcpy(indices_out, q.indices.data(), q.indices.size());
    for (std::size_t i = 0; i < q.scales.size(); ++i) scales_out[i] = q.scales[i].bits;
  });
}

size_t flute_canonical_words(int k, int n, int slice_bits) {
  return (static_cast<size_t>(k) * n * slice_bits + 31) / 32;
}

int flute_pack_canonical(const uint8_t* indices, int k, int n, int bits, const int* layout,
                         uint32_t* slice_hi, uint32_t* slice_lo) {
  return guard([&] {
    need(indices, "indices");
    need(slice_hi, "slice_hi");
    if (bits == 3) need(slice_lo, "slice_lo");
    QuantizedMatrix q;
    q.cfg.bits = bits;
    q.k = k;
    q.n = n;
    if (bits < 2 || bits > 4) throw ConfigError("bits must be in {2,3,4}");
    q.indices.assign(indices, indices + static_cast<size_t>(k) * n);
    const PackedWeights pw = reorder_and_split(q, to_layout(layout));
    std::memcpy(slice_hi, pw.slices[0].words.data(), pw.slices[0].words.size() * 4);
    if (bits == 3) std::memcpy(slice_lo, pw.slices[1].words.data(), pw.slices[1].words.size() * 4);
  });
}

int flute_unpack_canonical(const uint32_t* slice_hi, const uint32_t* slice_lo, int k, int n,
                           int bits, const int* layout, uint8_t* indices_out) {
  return guard([&] {
    need(indices_out, "indices_out");
    const LayoutDescriptor L = to_layout(layout);
    L.validate();
    const std::vector<uint8_t> idx = unpack_matrix(canonical_from(slice_hi, slice_lo, k, n, bits, L));
    std::memcpy(indices_out, idx.data(), idx.size());
  });
}

int flute_device_sizes(int k, int n, int bits, int group, size_t* weight_bytes,
                       size_t* scale_bytes) {
  return guard([&] {
    const DeviceGeometry g = device_geometry(k, n, bits, group);
    if (weight_bytes) *weight_bytes = g.weight_bytes();
    if (scale_bytes) *scale_bytes = g.scale_bytes();
  });
}

int flute_pack_device(const uint8_t* indices, int k, int n, int bits, int group, uint8_t* out) {
  return guard([&] {
    need(indices, "indices");
    need(out, "out");
    const std::vector<uint8_t> idx(indices, indices + static_cast<size_t>(k) * n);
    const std::vector<uint8_t> dev = pack_device(idx, k, n, bits, group);
    std::memcpy(out, dev.data(), dev.size());
  });
}

int flute_repack_canonical(const uint32_t* slice_hi, const uint32_t* slice_lo, int k, int n,
                           int bits, const int* layout, int group, uint8_t* out) {
  return guard([&] {
    need(out, "out");
    const LayoutDescriptor L = to_layout(layout);
    L.validate();
    const std::vector<uint8_t> dev =
        pack_device_from_canonical(canonical_from(slice_hi, slice_lo, k, n, bits, L), group);
    std::memcpy(out, dev.data(), dev.size());
  });
}

int flute_unpack_device(const uint8_t* packed, int k, int n, int bits, int group,
                        uint8_t* indices_out) {
  return guard([&] {
    need(packed, "packed");
    need(indices_out, "indices_out");
    const DeviceGeometry g = device_geometry(k, n, bits, group);
    const std::vector<uint8_t> dev(packed, packed + g.weight_bytes());
    const std::vector<uint8_t> idx = unpack_device(dev, k, n, bits, group);
    std::memcpy(indices_out, idx.data(), idx.size());
  });
}

int flute_scales_device(const uint16_t* scales, int k, int n, int group, uint16_t* out) {
  return guard([&] {
    need(scales, "scales");
    need(out, "out");
    QuantConfig{4, group}.validate(k);
    std::vector<Half> s(static_cast<size_t>(k / group) * n);
    for (size_t i = 0; i < s.size(); ++i) s[i] = Half::from_bits(scales[i]);
    const std::vector<uint16_t> d = scales_to_device(s, k, n, group);
    std::memcpy(out, d.data(), d.size() * 2);
  });
}

int flute_vlut_build(const float* table_values, int bits, int dup, uint32_t* out) {
  return guard([&] {
    need(table_values, "table_values");
    need(out, "out");
    LookupTable t;
    t.bits = bits;
    if (bits < 1 || bits > 4) throw ConfigError("bits must be in {2,3,4}");
    t.values.assign(table_values, table_values + (1 << bits));
    const VectorizedTable vt = make_vectorized_lut(t, dup);
    for (std::size_t e = 0; e < vt.entries.size(); ++e) {
      const uint32_t wv = static_cast<uint32_t>(vt.entries[e].first.bits) |
                          (static_cast<uint32_t>(vt.entries[e].second.bits) << 16);
      for (int c = 0; c < dup; ++c) out[vt.address(static_cast<uint32_t>(e), c)] = wv;
    }
  });
}

int flute_vlut_device_words(const uint32_t* vlut_words, int bits, uint32_t* out) {
  return guard([&] {
    need(out, "out");
    const std::vector<uint32_t> d = device_vlut_words(table_from_words(vlut_words, bits));
    std::memcpy(out, d.data(), d.size() * 4);
  });
}

int flute_vec_dequantize(uint32_t pair, uint16_t scale, const uint32_t* vlut_words, int bits,
                         uint32_t* out) {
  return guard([&] {
    need(out, "out");
    const auto r = vec_dequantize(pair, Half::from_bits(scale), table_from_words(vlut_words, bits));
    *out = static_cast<uint32_t>(r.first.bits) | (static_cast<uint32_t>(r.second.bits) << 16);
  });
}

int flute_plan_stream_k(int tiles_m, int tiles_n, int tiles_k, int workers, int64_t* ranges,
                        int64_t* fixups, int max_fixups, int* n_fixups, int64_t* total_slots) {
  return guard([&] {
    need(ranges, "ranges");
    const StreamKPlan p = plan_stream_k(TileGrid{tiles_m, tiles_n, tiles_k}, workers);
    for (int w = 0; w < workers; ++w) {
      ranges[2 * w] = p.ranges[w].begin;
      ranges[2 * w + 1] = p.ranges[w].end;
    }
    if (n_fixups) *n_fixups = static_cast<int>(p.fixups.size());
    if (total_slots) *total_slots = p.total_slots;
    if (fixups) {
      for (int f = 0; f < static_cast<int>(p.fixups.size()) && f < max_fixups; ++f) {
        fixups[4 * f] = p.fixups[f].tile;
        fixups[4 * f + 1] = p.fixups[f].finisher;
        fixups[4 * f + 2] = p.fixups[f].slot_base;
        fixups[4 * f + 3] = static_cast<int64_t>(p.fixups[f].contributors.size());
      }
    }
  });
}

int flute_plan_traffic(int m, int k, int n, int bits, int group, const int* layout, int workers,
                       int stages, int tile_m, uint64_t* stats) {
  return guard([&] {
    need(stats, "stats");
    ProblemShape s;
    s.m = m;
    s.k = k;
    s.n = n;
    s.cfg = QuantConfig{bits, group};
    s.layout = to_layout(layout);
    s.workers = workers;
    s.stages = stages;
    s.tile_m = tile_m;
    const TrafficStats t = plan_traffic(s);
    const uint64_t v[7] = {t.bytes_weights,     t.bytes_scales, t.bytes_table, t.bytes_activations,
                           t.bytes_partials_rw, t.bytes_output, t.flops};
    std::memcpy(stats, v, sizeof(v));
  });
}

double flute_bits_per_param(int bits, int group) {
  try {
    return bits_per_param(QuantConfig{bits, group});
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return -1.0;
  }
}

int flute_device_count(void) { return flute_dev::device_count(); }

int flute_sm_count(int device) {
  int v = 0;
  if (guard([&] { v = flute_dev::sm_count(device); }) != FLUTE_OK) return -1;
  return v;
}

int flute_max_workers(int m) {
  int v = -1;
  if (guard([&] { v = flute_dev::max_workers(m, 4); }) != FLUTE_OK) return -1;
  return v;
}

int flute_default_workers(int m, int k, int n, int bits) {
  int v = -1;
  if (guard([&] { v = flute_dev::default_workers(m, k, n, bits); }) != FLUTE_OK) return -1;
  return v;
}

size_t flute_workspace_bytes(int m, int workers) { return flute_dev::workspace_bytes(m, workers); }

int flute_qgemm(const void* x, int m, int k, int n, const void* w, const void* scales,
                const void* vlut, int bits, int group, void* y, void* workspace,
                size_t workspace_bytes, int workers, void* stream) {
  return guard([&] {
    QuantConfig{bits, group}.validate(k);
    flute_dev::GemmArgs a;
    a.x = x;
    a.m = m;
    a.k = k;
    a.n = n;
    a.w = w;
    a.scales = scales;
    a.vlut = vlut;
    a.bits = bits;
    a.group = group;
    a.y = y;
    a.workspace = workspace;
    a.workspace_bytes = workspace_bytes;
    a.workers = workers;
    a.stream = stream;
    flute_dev::qgemm(a);
  });
}

int flute_weights_create(const uint8_t* packed_host, const uint16_t* scales_dev_layout_host,
                         const uint32_t* vlut_words, int k, int n, int bits, int group,
                         flute_weights** out) {
  return guard([&] {
    need(packed_host, "packed_host");
    need(scales_dev_layout_host, "scales");
    need(out, "out");
    const DeviceGeometry g = device_geometry(k, n, bits, group);
    // Recover indices + [n][k/g] scales from the device layouts, then reuse
    // the DeviceWeights constructor (keeps one upload path).
    const std::vector<uint8_t> idx =
        unpack_device(std::vector<uint8_t>(packed_host, packed_host + g.weight_bytes()), k, n, bits, group);
    const int gpc = k / group, gp = g.groups_padded();
    std::vector<Half> sc(static_cast<size_t>(gpc) * n);
    for (int col = 0; col < n; ++col) {
      const int nt = col / kUnitN, c = col % kUnitN;
      const int j = c / 16, gr = c % 8, h = (c % 16) / 8;
      for (int G = 0; G < gpc; ++G)
        sc[static_cast<size_t>(col) * gpc + G] = Half::from_bits(
            scales_dev_layout_host[(static_cast<size_t>(nt) * gp + G) * kUnitN + gr * 8 + j * 2 + h]);
    }
    const VectorizedTable vt = table_from_words(vlut_words, bits);
    LookupTable t;
    t.bits = bits;
    for (int i = 0; i < (1 << bits); ++i) t.values.push_back(f16_to_f32(vt.entries[static_cast<size_t>(i) << bits].first));
    auto* h = new flute_weights;
    h->impl = new DeviceWeights(idx, sc, t, k, n, QuantConfig{bits, group});
    h->k = k;
    h->n = n;
    h->bits = bits;
    h->group = group;
    *out = h;
  });
}

int flute_weights_from_indices(const uint8_t* indices, const uint16_t* scales,
                               const float* table_values, int k, int n, int bits, int group,
                               flute_weights** out) {
  return guard([&] {
    need(indices, "indices");
    need(scales, "scales");
    need(table_values, "table_values");
    need(out, "out");
    QuantConfig{bits, group}.validate(k);
    std::vector<Half> sc(static_cast<size_t>(k / group) * n);
    for (size_t i = 0; i < sc.size(); ++i) sc[i] = Half::from_bits(scales[i]);
    LookupTable t;
    t.bits = bits;
    t.values.assign(table_values, table_values + (1 << bits));
    auto* h = new flute_weights;
    try {
      h->impl = new DeviceWeights(std::vector<uint8_t>(indices, indices + static_cast<size_t>(k) * n),
                                  sc, t, k, n, QuantConfig{bits, group});
    } catch (...) {
      delete h;
      throw;
    }
    h->k = k;
    h->n = n;
    h->bits = bits;
    h->group = group;
    *out = h;
  });
}

namespace {
flute_weights* wrap(std::unique_ptr<DeviceWeights> dw, int k, int n, int bits, int group) {
  auto* h = new flute_weights;
  h->impl = dw.release();
  h->k = k;
  h->n = n;
  h->bits = bits;
  h->group = group;
  return h;
}
}  // namespace

int flute_quantize_device(const float* w_dev, int k, int n, int bits, int group, uint8_t* idx_dev,
                          uint16_t* scales_dev, void* stream) {
  return guard([&] { quantize_on_device(w_dev, k, n, QuantConfig{bits, group}, idx_dev, scales_dev, stream); });
}

int flute_weights_from_device(const uint8_t* idx_dev, const uint16_t* scales_dev,
                              const uint16_t* table16, int k, int n, int bits, int group,
                              void* stream, flute_weights** out) {
  return guard([&] {
    need(table16, "table16");
    need(out, "out");
    if (bits < 2 || bits > 4) throw ConfigError("bits must be in {2,3,4}");
    std::vector<Half> t(std::size_t{1} << bits);
    for (std::size_t i = 0; i < t.size(); ++i) t[i] = Half::from_bits(table16[i]);
    *out = wrap(DeviceWeights::from_device_indices(idx_dev, scales_dev, t, k, n, QuantConfig{bits, group},
                                                   stream),
                k, n, bits, group);
  });
}

namespace {
MatF host_matrix(const float* p, int rows, int cols, const char* what) {
  need(p, what);
  if (rows < 1 || cols < 1) throw ConfigError(std::string(what) + ": dimensions must be positive");
  MatF m(rows, cols);
  std::memcpy(m.data.data(), p, static_cast<std::size_t>(rows) * cols * sizeof(float));
  return m;
}
}  // namespace

int flute_ste_evaluate(const float* w, const float* x, int m, int k, int n, int bits, int group,
                       const double* sigma, double* loss, double* grad, uint8_t* idx) {
  return guard([&] {
    need(sigma, "sigma");
    need(loss, "loss");
    const MatF W = host_matrix(w, k, n, "w");
    const MatF X = host_matrix(x, m, k, "x");
    const QuantConfig cfg{bits, group};
    cfg.validate(k);
    const std::size_t groups = static_cast<std::size_t>(k / group) * n;
    const SteEval e = ste_evaluate(W, X, cfg, std::span<const double>(sigma, groups));
    *loss = e.loss;
    if (grad) std::memcpy(grad, e.grad.data(), groups * sizeof(double));
    if (idx) std::memcpy(idx, e.indices.data(), e.indices.size());
  });
}

int flute_refine_scales(const float* w, const float* x, int m, int k, int n, int bits, int group,
                        int steps, double lr, uint8_t* idx, uint16_t* scales, double* sigma,
                        double* losses, int* failed_step) {
  if (failed_step) *failed_step = -1;
  return guard([&] {
    need(idx, "idx");
    need(scales, "scales");
    const MatF W = host_matrix(w, k, n, "w");
    const MatF X = host_matrix(x, m, k, "x");
    RefineResult r;
    try {
      r = refine_scales(W, X, QuantConfig{bits, group}, steps, lr);
    } catch (const OptimizationError& e) {
      if (failed_step) *failed_step = e.step;
      throw;
    }
    std::memcpy(idx, r.quantized.indices.data(), r.quantized.indices.size());
    for (std::size_t g = 0; g < r.quantized.scales.size(); ++g) scales[g] = r.quantized.scales[g].bits;
    if (sigma) std::memcpy(sigma, r.sigma_tilde.data(), r.sigma_tilde.size() * sizeof(double));
    if (losses) {
      losses[0] = r.initial_loss;
      losses[1] = r.final_loss;
    }
  });
}

int flute_flte_info(const uint8_t* bytes, size_t len, int* bits, int* group, int* k, int* n) {
  return guard([&] {
    need(bytes, "bytes");
    const FlteModel m = parse_flte(bytes, len);
    if (bits) *bits = m.cfg.bits;
    if (group) *group = m.cfg.group_size;
    if (k) *k = m.k;
    if (n) *n = m.n;
  });
}

int flute_weights_from_flte(const uint8_t* bytes, size_t len, void* stream, flute_weights** out) {
  return guard([&] {
    need(bytes, "bytes");
    need(out, "out");
    const FlteModel m = parse_flte(bytes, len);
    *out = wrap(DeviceWeights::from_flte(m, stream), m.k, m.n, m.cfg.bits, m.cfg.group_size);
  });
}

int flute_flte_write(const uint8_t* indices, const uint16_t* scales, const float* table_values,
                     int k, int n, int bits, int group, const int* layout, uint8_t* out, size_t cap,
                     size_t* len) {
  return guard([&] {
    need(indices, "indices");
    need(scales, "scales");
    need(table_values, "table_values");
    need(len, "len");
    QuantizedMatrix q;
    q.cfg = QuantConfig{bits, group};
    q.cfg.validate(k);
    q.k = k;
    q.n = n;
    q.indices.assign(indices, indices + static_cast<size_t>(k) * n);
    q.scales.resize(static_cast<size_t>(k / group) * n);
    for (size_t i = 0; i < q.scales.size(); ++i) q.scales[i] = Half::from_bits(scales[i]);
    q.table.bits = bits;
    q.table.values.assign(table_values, table_values + (1 << bits));
    const PackedWeights pw = reorder_and_split(q, to_layout(layout));
    const std::vector<uint8_t> b = flte_bytes(make_flte_model(q, pw));
    *len = b.size();
    if (out != nullptr) {
      if (cap < b.size()) throw InputError("flte_write: output buffer too small");
      std::memcpy(out, b.data(), b.size());
    }
  });
}

int flute_weights_destroy(flute_weights* w) {
  return guard([&] {
    if (w == nullptr) return;
    delete w->impl;
    delete w;
  });
}

int flute_weights_info(const flute_weights* w, int* k, int* n, int* bits, int* group) {
  return guard([&] {
    need(w, "weights");
    if (k) *k = w->k;
    if (n) *n = w->n;
    if (bits) *bits = w->bits;
    if (group) *group = w->group;
  });
}

int flute_weights_autotune(flute_weights* w, int m, void* stream, char* report, size_t cap) {
  return guard([&] {
    need(w, "weights");
    const std::string r = w->impl->autotune(m, stream);
    if (report && cap > 0) std::snprintf(report, cap, "%s", r.c_str());
  });
}

int flute_weights_reserve(flute_weights* w, int max_m) {
  return guard([&] {
    need(w, "weights");
    if (max_m < 1) throw ConfigError("reserve: max_m must be >= 1");
    w->impl->reserve(max_m);
  });
}

int flute_gemm(flute_weights* w, const void* x_dev, int m, void* y_dev, int workers,
               void* stream) {
  return guard([&] {
    need(w, "weights");
    w->impl->gemm(static_cast<const Half*>(x_dev), m, static_cast<Half*>(y_dev), workers, stream);
  });
}

int flute_gemm_host_batch(flute_weights* const* ws, const uint16_t* const* x_host, const int* m,
                          uint16_t* const* y_host, int count, int workers, void* stream) {
  return guard([&] {
    if (count > 0) {
      need(ws, "weights");
      need(x_host, "x_host");
      need(m, "m");
      need(y_host, "y_host");
    }
    std::vector<DeviceWeights*> h(static_cast<std::size_t>(std::max(count, 0)));
    for (int i = 0; i < count; ++i) {
      need(ws[i], "weights[i]");
      h[i] = ws[i]->impl;
    }
    DeviceWeights::gemm_host_batch(h.data(), x_host, m, y_host, count, workers, stream);
  });
}

struct flute_host_batch {
  HostBatch* impl = nullptr;
};

int flute_host_batch_create(flute_weights* const* ws, const uint16_t* const* x_host, const int* m,
                            uint16_t* const* y_host, int count, int workers,
                            flute_host_batch** out) {
  return guard([&] {
    need(out, "out");
    if (count > 0) {
      need(ws, "weights");
      need(x_host, "x_host");
      need(m, "m");
      need(y_host, "y_host");
    }
    std::vector<DeviceWeights*> h(static_cast<std::size_t>(std::max(count, 0)));
    for (int i = 0; i < count; ++i) {
      need(ws[i], "weights[i]");
      h[i] = ws[i]->impl;
    }
    auto* b = new flute_host_batch();
    try {
      b->impl = new HostBatch(h.data(), x_host, m, y_host, count, workers);
    } catch (...) {
      delete b;
      throw;
    }
    *out = b;
  });
}

int flute_host_batch_run(flute_host_batch* b, void* stream) {
  return guard([&] {
    need(b, "batch");
    b->impl->run(stream);
  });
}

void flute_host_batch_destroy(flute_host_batch* b) {
  if (!b) return;
  delete b->impl;
  delete b;
}

int flute_gemm_host(flute_weights* w, const uint16_t* x_host, int m, uint16_t* y_host,
                    int workers, void* stream) {
  return guard([&] {
    need(w, "weights");
    need(x_host, "x_host");
    need(y_host, "y_host");
    w->impl->gemm_host_raw(x_host, m, y_host, workers, stream);
  });
}

int flute_execute(const uint16_t* x, int m, const uint32_t* slice_hi, const uint32_t* slice_lo,
                  int k, int n, int bits, int group, const int* layout, const uint16_t* scales,
                  const uint32_t* vlut_words, int dup, int workers, int stages, int tile_m,
                  uint16_t* y, uint64_t* stats) {
  return guard([&] {
    need(x, "x");
    need(scales, "scales");
    need(vlut_words, "vlut_words");
    need(y, "y");
    if (m < 1) throw ConfigError("matmul: m must be >= 1");
    if (dup < 1) throw ConfigError("vectorized table: dup must be >= 1");
    const PackedWeights pw = canonical_from(slice_hi, slice_lo, k, n, bits, to_layout(layout));
    // entry e, copy 0 lives at e * dup (vec_lut.hpp:18-30)
    std::vector<uint32_t> words(std::size_t{1} << (2 * bits));
    for (std::size_t e = 0; e < words.size(); ++e) words[e] = vlut_words[e * dup];
    VectorizedTable lut = table_from_words(words.data(), bits);
    MatH xm(m, k);
    std::memcpy(static_cast<void*>(xm.data.data()), x, xm.data.size() * 2);
    std::vector<Half> sc(static_cast<std::size_t>(k) * n / std::max(group, 1));
    std::memcpy(static_cast<void*>(sc.data()), scales, sc.size() * 2);
    MatmulProblem p;
    p.x = &xm;
    p.weights = &pw;
    p.scales = &sc;
    p.lut = &lut;
    p.cfg = QuantConfig{bits, group};
    p.workers = workers;
    p.stages = stages;
    p.tile_m = tile_m;
    const MatmulResult r = execute(p);
    std::memcpy(y, r.y.data.data(), r.y.data.size() * 2);
    if (stats) {
      const TrafficStats& t = r.stats;
      const uint64_t v[7] = {t.bytes_weights, t.bytes_scales, t.bytes_table, t.bytes_activations,
                             t.bytes_partials_rw, t.bytes_output, t.flops};
      std::memcpy(stats, v, sizeof v);
    }
  });
}

int flute_shard_range(int k, int n, int bits, int group, int world, int rank, int* n0, int* n1,
                      size_t* w_off, size_t* w_bytes, size_t* s_off, size_t* s_bytes) {
  return guard([&] {
    const ShardRange r = shard_range(k, n, bits, group, world, rank);
    if (n0) *n0 = r.n0;
    if (n1) *n1 = r.n1;
    if (w_off) *w_off = r.w_off;
    if (w_bytes) *w_bytes = r.w_bytes;
    if (s_off) *s_off = r.s_off;
    if (s_bytes) *s_bytes = r.s_bytes;
  });
}

int flute_qgemm_peers(const void* x, int m, int k, int n, const void* w, const void* scales,
                      const void* vlut, int bits, int group, void* const* y_peers, int n_peers,
                      int ldy, int ycol0, void* workspace, size_t workspace_bytes, int workers,
                      void* stream) {
  return guard([&] {
    flute_dev::GemmArgs a;
    a.x = x;
    a.m = m;
    a.k = k;
    a.n = n;
    a.w = w;
    a.scales = scales;
    a.vlut = vlut;
    a.bits = bits;
    a.group = group;
    a.y_peers = y_peers;
    a.n_peers = n_peers;
    a.ldy = ldy;
    a.ycol0 = ycol0;
    a.workspace = workspace;
    a.workspace_bytes = workspace_bytes;
    a.workers = workers;
    a.stream = stream;
    if (n_peers < 1) throw ConfigError("qgemm_peers: need at least one output buffer");
    flutesim::QuantConfig{bits, group}.validate(k);
    flute_dev::qgemm(a);
  });
}

int flute_gemm_peers(flute_weights* w, const void* x_dev, int m, void* const* y_peers, int n_peers,
                     int ldy, int ycol0, int workers, void* stream) {
  return guard([&] {
    need(w, "weights");
    w->impl->gemm_peers(static_cast<const Half*>(x_dev), m, y_peers, n_peers, ldy, ycol0, workers,
                        stream);
  });
}

int flute_comm_unique_id(uint8_t* id_out) {
  return guard([&] {
    need(id_out, "id_out");
    const std::vector<uint8_t> id = Communicator::unique_id();
    std::memcpy(id_out, id.data(), id.size());
  });
}

int flute_comm_create(const uint8_t* id, int world, int rank, flute_comm** out) {
  return guard([&] {
    need(out, "out");
    *out = nullptr;
    auto c = std::make_unique<flute_comm>();
    c->impl = std::make_unique<Communicator>(id, world, rank);
    *out = c.release();
  });
}

int flute_comm_destroy(flute_comm* c) {
  return guard([&] { delete c; });
}

int flute_sharded_create(flute_comm* c, const uint8_t* indices, const uint16_t* scales,
                         const float* table_values, int k, int n, int bits, int group, int max_m,
                         flute_sharded** out) {
  return guard([&] {
    need(c, "comm");
    need(indices, "indices");
    need(scales, "scales");
    need(table_values, "table_values");
    need(out, "out");
    *out = nullptr;
    const QuantConfig cfg{bits, group};
    cfg.validate(k);
    if (n < 1) throw ConfigError("n must be >= 1");
    std::vector<uint8_t> idx(indices, indices + static_cast<size_t>(k) * n);
    const size_t ns = static_cast<size_t>(n) * (k / group);
    std::vector<Half> sc(ns);
    for (size_t i = 0; i < ns; ++i) sc[i] = Half::from_bits(scales[i]);
    LookupTable t;
    t.bits = bits;
    t.values.assign(table_values, table_values + (size_t{1} << bits));
    auto s = std::make_unique<flute_sharded>();
    s->impl = std::make_unique<ShardedWeights>(*c->impl, idx, sc, t, k, n, cfg, max_m);
    *out = s.release();
  });
}

int flute_sharded_destroy(flute_sharded* s) {
  return guard([&] { delete s; });
}

int flute_sharded_info(const flute_sharded* s, int* n0, int* n1) {
  return guard([&] {
    need(s, "sharded");
    if (n0) *n0 = s->impl->n0();
    if (n1) *n1 = s->impl->n1();
  });
}

int flute_sharded_gemm(flute_sharded* s, const void* x_dev, int m, void* y_dev, void* stream) {
  return guard([&] {
    need(s, "sharded");
    s->impl->gemm(static_cast<const Half*>(x_dev), m, static_cast<Half*>(y_dev), stream);
  });
}

int flute_sharded_gemm_fused(flute_sharded* s, const void* x_dev, int m, const void** y_out,
                             void* stream) {
  return guard([&] {
    need(s, "sharded");
    need(y_out, "y_out");
    *y_out = s->impl->gemm_fused(static_cast<const Half*>(x_dev), m, stream);
  });
}

int flute_dequant_all_device(const uint32_t* vlut_words, int bits, const uint16_t* scales,
                             int n_scales, uint32_t* out_host) {
  return guard([&] {
    need(scales, "scales");
    need(out_host, "out_host");
    const std::vector<uint32_t> d = device_vlut_words(table_from_words(vlut_words, bits));
    flute_dev::dequant_all(d.data(), bits, scales, n_scales, out_host);
  });
}

int flute_debug_times(uint64_t* out, int workers) {
  return guard([&] {
    need(out, "out");
    flute_dev::debug_times(reinterpret_cast<unsigned long long*>(out), workers);
  });
}

int flute_mma_fragment(const uint16_t* a, const uint16_t* b, float* c, int m, int n, int k) {
  return guard([&] {
    need(a, "a");
    need(b, "b");
    need(c, "c");
    FragDims d{m, n, k};
    mma_fragment(std::span<const Half>(reinterpret_cast<const Half*>(a), static_cast<size_t>(m) * k),
                 std::span<const Half>(reinterpret_cast<const Half*>(b), static_cast<size_t>(k) * n),
                 std::span<float>(c, static_cast<size_t>(m) * n), d);
  });
}

}  // extern "C"
