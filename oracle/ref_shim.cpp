// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// extern "C" shim over the *unmodified* reference library (flutesim, compiled
// from /root/reference/proj/src by oracle/Makefile into oracle/_ref/).  It lets
// the Python tests, the golden-fixture generator and bench.py's reference arm
// drive the reference's own code path through ctypes with plain pointers.
//
// Entry points mirror the reference API they wrap:
//   fref_nf_table        -> build_nf_table            (nf_table.cpp:95)
//   fref_quantize        -> quantize_matrix           (quantize.cpp:81)
//   fref_pack            -> reorder_and_split         (pack.cpp:83)
//   fref_unpack          -> unpack_matrix             (pack.cpp:156)
//   fref_packed_pos      -> packed_pos                (pack.cpp:48)
//   fref_vlut            -> make_vectorized_lut       (vec_lut.cpp:10)
//   fref_vec_dequantize  -> vec_dequantize            (vec_lut.cpp:39)
//   fref_plan_stream_k   -> plan_stream_k             (streamk.cpp:17)
//   fref_execute         -> execute                   (engine.cpp:345)
//   fref_plan_traffic    -> plan_traffic              (engine.cpp:389)
//   fref_f32_to_f16 / fref_f16_to_f32 -> half.hpp:81-87
//   fref_flte_write      -> quantize + reorder_and_split + make_flte_model + write_flte (flte.cpp:80-118)
//   fref_flte_parse      -> read_flte (flte.cpp:120-213): section / offset of a ParseError
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include <sstream>

#include "flutesim/engine.hpp"
#include "flutesim/flte.hpp"
#include "flutesim/errors.hpp"
#include "flutesim/half.hpp"
#include "flutesim/nf_table.hpp"
#include "flutesim/pack.hpp"
#include "flutesim/quantize.hpp"
#include "flutesim/streamk.hpp"
#include "flutesim/vec_lut.hpp"

using namespace flutesim;

namespace {
thread_local std::string g_err;

// 0 ok, 1 ConfigError, 2 InputError, 3 InternalError, 4 anything else.
template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const ConfigError& e) {
    g_err = e.what();
    return 1;
  } catch (const InputError& e) {
    g_err = e.what();
    return 2;
  } catch (const InternalError& e) {
    g_err = e.what();
    return 3;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 4;
  }
}

LayoutDescriptor layout_from(const int* l) {
  LayoutDescriptor d;
  d.tile_m = l[0];
  d.tile_n = l[1];
  d.tile_k = l[2];
  d.frag_m = l[3];
  d.frag_n = l[4];
  d.frag_k = l[5];
  return d;
}

PackedWeights packed_from(int k, int n, int bits, const int* layout,
                          const std::uint32_t* s0, const std::uint32_t* s1) {
  PackedWeights pw;
  pw.layout = layout_from(layout);
  pw.bits = bits;
  pw.k = k;
  pw.n = n;
  const std::size_t total = static_cast<std::size_t>(k) * n;
  if (bits == 3) {
    pw.slices = {BitSlice{2, {}}, BitSlice{1, {}}};
    pw.slices[0].words.assign(s0, s0 + (total * 2 + 31) / 32);
    pw.slices[1].words.assign(s1, s1 + (total + 31) / 32);
  } else {
    pw.slices = {BitSlice{bits, {}}};
    pw.slices[0].words.assign(s0, s0 + (total * bits + 31) / 32);
  }
  return pw;
}
}  // namespace

extern "C" {

const char* fref_last_error() { return g_err.c_str(); }

int fref_flte_write(const float* w, int k, int n, int bits, int group, const int* layout,
                    std::uint8_t* out, std::size_t cap, std::size_t* len) {
  return guarded([&] {
    MatF m(k, n);
    std::memcpy(m.data.data(), w, sizeof(float) * m.data.size());
    const QuantizedMatrix q = quantize_matrix(m, QuantConfig{bits, group});
    const LayoutDescriptor L{layout[0], layout[1], layout[2], layout[3], layout[4], layout[5]};
    const PackedWeights pw = reorder_and_split(q, L);
    std::ostringstream os(std::ios::binary);
    write_flte(os, make_flte_model(q, pw));
    const std::string b = os.str();
    *len = b.size();
    if (out) {
      if (cap < b.size()) throw InputError("buffer too small");
      std::memcpy(out, b.data(), b.size());
    }
  });
}

// 0 = parsed; 5 = ParseError (section copied to sec_out, offset to *off);
// other codes as guarded().
int fref_flte_parse(const std::uint8_t* bytes, std::size_t len, char* sec_out, std::size_t sec_cap,
                    std::size_t* off) {
  try {
    std::istringstream is(std::string(reinterpret_cast<const char*>(bytes), len), std::ios::binary);
    (void)read_flte(is);
    return 0;
  } catch (const ParseError& e) {
    g_err = e.what();
    std::snprintf(sec_out, sec_cap, "%s", e.section.c_str());
    *off = e.offset;
    return 5;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 4;
  }
}

std::uint16_t fref_f32_to_f16(float x) { return f32_to_f16(x).to_bits(); }
float fref_f16_to_f32(std::uint16_t h) { return f16_to_f32(Half::from_bits(h)); }

int fref_nf_table(int bits, float* values_out) {
  return guarded([&] {
    const LookupTable t = build_nf_table(bits);
    std::memcpy(values_out, t.values.data(), t.values.size() * sizeof(float));
  });
}

// w: k x n row-major f32.  idx_out: k*n u8.  scales_out: (k*n/group) u16.
int fref_quantize(const float* w, int k, int n, int bits, int group,
                  std::uint8_t* idx_out, std::uint16_t* scales_out) {
  return guarded([&] {
    MatF m(k, n);
    std::memcpy(m.data.data(), w, sizeof(float) * static_cast<std::size_t>(k) * n);
    const QuantizedMatrix q = quantize_matrix(m, QuantConfig{bits, group});
    std::memcpy(idx_out, q.indices.data(), q.indices.size());
    for (std::size_t i = 0; i < q.scales.size(); ++i) scales_out[i] = q.scales[i].to_bits();
  });
}

// Words per slice: slice0 ceil(k*n*w0/32), slice1 (3-bit only) ceil(k*n/32).
int fref_pack(const std::uint8_t* idx, int k, int n, int bits, const int* layout,
              std::uint32_t* slice0, std::uint32_t* slice1) {
  return guarded([&] {
    QuantizedMatrix q;
    q.cfg.bits = bits;
    q.cfg.group_size = 32;
    q.k = k;
    q.n = n;
    q.indices.assign(idx, idx + static_cast<std::size_t>(k) * n);
    const PackedWeights pw = reorder_and_split(q, layout_from(layout));
    std::memcpy(slice0, pw.slices[0].words.data(), pw.slices[0].words.size() * 4);
    if (pw.slices.size() > 1) {
      std::memcpy(slice1, pw.slices[1].words.data(), pw.slices[1].words.size() * 4);
    }
  });
}

int fref_unpack(int k, int n, int bits, const int* layout, const std::uint32_t* s0,
                const std::uint32_t* s1, std::uint8_t* idx_out) {
  return guarded([&] {
    const PackedWeights pw = packed_from(k, n, bits, layout, s0, s1);
    const std::vector<std::uint8_t> out = unpack_matrix(pw);
    std::memcpy(idx_out, out.data(), out.size());
  });
}

long long fref_packed_pos(const int* layout, int k, int n, int i, int j) {
  return static_cast<long long>(packed_pos(layout_from(layout), k, n, i, j));
}

// out: 2^(2b) u32 words, low half = first (even k), high half = second.
int fref_vlut(const float* values, int bits, int dup, std::uint32_t* out) {
  return guarded([&] {
    LookupTable t;
    t.bits = bits;
    t.values.assign(values, values + (1 << bits));
    const VectorizedTable vt = make_vectorized_lut(t, dup);
    for (std::size_t e = 0; e < vt.entries.size(); ++e) {
      out[e] = static_cast<std::uint32_t>(vt.entries[e].first.to_bits()) |
               (static_cast<std::uint32_t>(vt.entries[e].second.to_bits()) << 16);
    }
  });
}

int fref_vec_dequantize(const float* values, int bits, std::uint32_t pair,
                        std::uint16_t scale, std::uint32_t* out) {
  return guarded([&] {
    LookupTable t;
    t.bits = bits;
    t.values.assign(values, values + (1 << bits));
    const VectorizedTable vt = make_vectorized_lut(t, 1);
    const auto r = vec_dequantize(pair, Half::from_bits(scale), vt);
    *out = static_cast<std::uint32_t>(r.first.to_bits()) |
           (static_cast<std::uint32_t>(r.second.to_bits()) << 16);
  });
}

// ranges_out: 2*workers longs.  fixups_out (may be null): per split tile
// {tile, finisher, slot_base, n_contrib}; returns the count via *n_fixups.
int fref_plan_stream_k(int tm, int tn, int tk, int workers, long long* ranges_out,
                       long long* fixups_out, int max_fixups, int* n_fixups,
                       long long* total_slots) {
  return guarded([&] {
    const StreamKPlan p = plan_stream_k(TileGrid{tm, tn, tk}, workers);
    for (int w = 0; w < workers; ++w) {
      ranges_out[2 * w] = p.ranges[w].begin;
      ranges_out[2 * w + 1] = p.ranges[w].end;
    }
    *n_fixups = static_cast<int>(p.fixups.size());
    *total_slots = p.total_slots;
    if (fixups_out != nullptr) {
      for (int f = 0; f < static_cast<int>(p.fixups.size()) && f < max_fixups; ++f) {
        fixups_out[4 * f] = p.fixups[f].tile;
        fixups_out[4 * f + 1] = p.fixups[f].finisher;
        fixups_out[4 * f + 2] = p.fixups[f].slot_base;
        fixups_out[4 * f + 3] = static_cast<long long>(p.fixups[f].contributors.size());
      }
    }
  });
}

// Full reference execute.  x: m x k f16 bits; scales: k*n/group f16 bits;
// table values: 2^bits f32 (narrowed by make_vectorized_lut as the reference
// does).  y_out: m x n f16 bits.  stats_out: 7 u64 (weights, scales, table,
// activations, partials_rw, output, flops).  mode: 0 serial, 1 parallel.
int fref_execute(const std::uint16_t* x, int m, int k, int n, int bits, int group,
                 const int* layout, const std::uint32_t* s0, const std::uint32_t* s1,
                 const std::uint16_t* scales, const float* table_values, int dup,
                 int workers, int stages, int tile_m, int mode, std::uint16_t* y_out,
                 std::uint64_t* stats_out) {
  return guarded([&] {
    MatH xm(m, k);
    for (std::size_t i = 0; i < xm.data.size(); ++i) xm.data[i] = Half::from_bits(x[i]);
    const PackedWeights pw = packed_from(k, n, bits, layout, s0, s1);
    std::vector<Half> sc(static_cast<std::size_t>(k) * n / group);
    for (std::size_t i = 0; i < sc.size(); ++i) sc[i] = Half::from_bits(scales[i]);
    LookupTable t;
    t.bits = bits;
    t.values.assign(table_values, table_values + (1 << bits));
    const VectorizedTable vt = make_vectorized_lut(t, dup);
    MatmulProblem p;
    p.x = &xm;
    p.weights = &pw;
    p.scales = &sc;
    p.lut = &vt;
    p.cfg = QuantConfig{bits, group};
    p.workers = workers;
    p.stages = stages;
    p.tile_m = tile_m;
    p.mode = mode == 0 ? ExecMode::kSerial : ExecMode::kParallel;
    const MatmulResult r = execute(p);
    for (std::size_t i = 0; i < r.y.data.size(); ++i) y_out[i] = r.y.data[i].to_bits();
    if (stats_out != nullptr) {
      stats_out[0] = r.stats.bytes_weights;
      stats_out[1] = r.stats.bytes_scales;
      stats_out[2] = r.stats.bytes_table;
      stats_out[3] = r.stats.bytes_activations;
      stats_out[4] = r.stats.bytes_partials_rw;
      stats_out[5] = r.stats.bytes_output;
      stats_out[6] = r.stats.flops;
    }
  });
}

int fref_plan_traffic(int m, int k, int n, int bits, int group, const int* layout,
                      int workers, int stages, int dup, int tile_m,
                      std::uint64_t* stats_out) {
  return guarded([&] {
    ProblemShape s;
    s.m = m;
    s.k = k;
    s.n = n;
    s.cfg = QuantConfig{bits, group};
    s.layout = layout_from(layout);
    s.workers = workers;
    s.stages = stages;
    s.dup = dup;
    s.tile_m = tile_m;
    const TrafficStats t = plan_traffic(s);
    stats_out[0] = t.bytes_weights;
    stats_out[1] = t.bytes_scales;
    stats_out[2] = t.bytes_table;
    stats_out[3] = t.bytes_activations;
    stats_out[4] = t.bytes_partials_rw;
    stats_out[5] = t.bytes_output;
    stats_out[6] = t.flops;
  });
}

// Learned-sigma refinement (quantize.cpp:141-282).  w: k x n, x: m x k
// row-major f32; sigma/grad [n][k/g] f64.  5 = OptimizationError (*step set).
int fref_ste_evaluate(const float* w, const float* x, int m, int k, int n, int bits, int group,
                      const double* sigma, double* loss, double* grad, std::uint8_t* idx) {
  return guarded([&] {
    MatF W(k, n), X(m, k);
    std::memcpy(W.data.data(), w, sizeof(float) * static_cast<std::size_t>(k) * n);
    std::memcpy(X.data.data(), x, sizeof(float) * static_cast<std::size_t>(m) * k);
    const std::size_t groups = static_cast<std::size_t>(k / group) * n;
    const SteEval e = ste_evaluate(W, X, QuantConfig{bits, group},
                                   std::span<const double>(sigma, groups));
    *loss = e.loss;
    std::memcpy(grad, e.grad.data(), groups * sizeof(double));
    std::memcpy(idx, e.indices.data(), e.indices.size());
  });
}

int fref_refine_scales(const float* w, const float* x, int m, int k, int n, int bits, int group,
                       int steps, double lr, std::uint8_t* idx, std::uint16_t* scales,
                       double* sigma, double* losses, int* step) {
  try {
    MatF W(k, n), X(m, k);
    std::memcpy(W.data.data(), w, sizeof(float) * static_cast<std::size_t>(k) * n);
    std::memcpy(X.data.data(), x, sizeof(float) * static_cast<std::size_t>(m) * k);
    const RefineResult r = refine_scales(W, X, QuantConfig{bits, group}, steps, lr);
    std::memcpy(idx, r.quantized.indices.data(), r.quantized.indices.size());
    for (std::size_t g = 0; g < r.quantized.scales.size(); ++g) scales[g] = r.quantized.scales[g].to_bits();
    std::memcpy(sigma, r.sigma_tilde.data(), r.sigma_tilde.size() * sizeof(double));
    losses[0] = r.initial_loss;
    losses[1] = r.final_loss;
    return 0;
  } catch (const OptimizationError& e) {
    g_err = e.what();
    *step = e.step;
    return 5;
  } catch (...) {
    return guarded([] { throw; });
  }
}

}  // extern "C"
