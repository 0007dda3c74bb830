// flute-b200 — host engine: the drop-in execute() (reference engine.cpp:345),
// the reference traffic model (engine.cpp:87-130, 375-418) and the
// device-resident weight handle.  All compute goes to the GPU kernel through
// flute_dev::qgemm; there is no CPU fallback.
#include <algorithm>
#include <string>
#include <vector>

#include "device_api.h"
#include "flutesim/engine.hpp"
#include "flutesim/flte.hpp"
#include "flutesim/nf_table.hpp"
#include "flutesim/errors.hpp"
#include "flutesim/mma.hpp"

namespace flutesim {

TrafficStats& TrafficStats::operator+=(const TrafficStats& o) {
  bytes_weights += o.bytes_weights;
  bytes_scales += o.bytes_scales;
  bytes_table += o.bytes_table;
  bytes_activations += o.bytes_activations;
  bytes_partials_rw += o.bytes_partials_rw;
  bytes_output += o.bytes_output;
  flops += o.flops;
  return *this;
}

namespace {

struct Shape {
  int m = 0, k = 0, n = 0, tile_m = 0;
  LayoutDescriptor L;
  QuantConfig cfg;
  TileGrid grid;
};

// engine.cpp:59-85 validation order and messages.
Shape make_shape(int m, int k, int n, const LayoutDescriptor& L, const QuantConfig& cfg,
                 int tile_m_override, int stages, int workers) {
  L.validate();
  cfg.validate(k);
  Shape s;
  s.m = m;
  s.k = k;
  s.n = n;
  s.L = L;
  s.cfg = cfg;
  s.tile_m = tile_m_override > 0 ? tile_m_override : L.tile_m;
  if (m < 1) throw ConfigError("matmul: m must be >= 1");
  if (workers < 1) throw ConfigError("matmul: workers must be >= 1");
  if (stages < 1) throw ConfigError("matmul: pipeline stages must be >= 1");
  if (s.tile_m % L.frag_m != 0) throw ConfigError("matmul: tile_m must divide by frag_m");
  if (k % L.tile_k != 0 || n % L.tile_n != 0) throw ConfigError("matmul: dims must divide by tile dims");
  s.grid = TileGrid{(m + s.tile_m - 1) / s.tile_m, n / L.tile_n, k / L.tile_k};
  return s;
}

int rows_in(const Shape& s, long mt) {
  return static_cast<int>(std::min<long>(s.tile_m, static_cast<long>(s.m) - mt * s.tile_m));
}

// The reference's per-worker accounting: every unit of a non-empty range is
// fetched once (activations, weights, scales), the table once per worker,
// partial tiles written by contributors and read by finishers, outputs once.
TrafficStats account(const Shape& s, int workers) {
  const StreamKPlan plan = plan_stream_k(s.grid, workers);
  const LayoutDescriptor& L = s.L;
  const std::uint64_t tile_bytes = static_cast<std::uint64_t>(s.tile_m) * L.tile_n * 2;
  const std::uint64_t unit_flops = static_cast<std::uint64_t>(s.tile_m / L.frag_m) *
                                   L.frags_per_tile_n() * L.frags_per_tile_k() * 2ull * L.frag_m *
                                   L.frag_n * L.frag_k;
  const std::uint64_t weight_tile = static_cast<std::uint64_t>(L.tile_elems()) * s.cfg.bits / 8;
  TrafficStats t;
  for (int w = 0; w < workers; ++w) {
    const WorkerRange r = plan.ranges[w];
    if (r.size() == 0) continue;
    t.bytes_table += (std::uint64_t{1} << (2 * s.cfg.bits)) * 4;
    for (long u = r.begin; u < r.end; ++u) {
      const long tile = u / s.grid.tiles_k;
      const long mt = tile / s.grid.tiles_n;
      const long kt = u % s.grid.tiles_k;
      t.bytes_activations += static_cast<std::uint64_t>(rows_in(s, mt)) * L.tile_k * 2;
      t.bytes_weights += weight_tile;
      const long k0 = kt * L.tile_k, k1 = k0 + L.tile_k - 1;
      t.bytes_scales +=
          static_cast<std::uint64_t>((k1 / s.cfg.group_size - k0 / s.cfg.group_size + 1) * L.tile_n) * 2;
      t.flops += unit_flops;
      const bool tile_end = u + 1 >= r.end || (u + 1) % s.grid.tiles_k == 0;
      if (!tile_end) continue;
      const bool finished = r.end >= (tile + 1) * s.grid.tiles_k;
      const bool started = r.begin <= tile * s.grid.tiles_k;
      if (!finished) {
        t.bytes_partials_rw += tile_bytes;
        continue;
      }
      if (!started) {
        t.bytes_partials_rw += tile_bytes * plan.fixup_for(tile)->contributors.size();
      }
      t.bytes_output += static_cast<std::uint64_t>(rows_in(s, mt)) * L.tile_n * 2;
    }
  }
  return t;
}

struct DeviceBuffer {
  void* p = nullptr;
  std::size_t bytes = 0;
  DeviceBuffer() = default;
  explicit DeviceBuffer(std::size_t n) : p(flute_dev::dev_alloc(n)), bytes(n) {}
  ~DeviceBuffer() { flute_dev::dev_free(p); }
  DeviceBuffer(const DeviceBuffer&) = delete;
  DeviceBuffer& operator=(const DeviceBuffer&) = delete;
  DeviceBuffer(DeviceBuffer&& o) noexcept : p(o.p), bytes(o.bytes) {
    o.p = nullptr;
    o.bytes = 0;
  }
  DeviceBuffer& operator=(DeviceBuffer&& o) noexcept {
    std::swap(p, o.p);
    std::swap(bytes, o.bytes);
    return *this;
  }
};

}  // namespace

// ---------------------------------------------------------------------------
// DeviceWeights
// ---------------------------------------------------------------------------

struct DeviceWeights::Impl {
  int k = 0, n = 0, bits = 0, group = 0;
  DeviceBuffer w, sc, lut, ws, ws_tc, xbuf, ybuf;
  // Buffers replaced by a larger one.  A HostBatch graph captured earlier may
  // still point at them, so they are kept until the handle is destroyed (a
  // handle must outlive its batches) instead of being freed on growth.
  std::vector<DeviceBuffer> retired;

  // replace `b` by a fresh (zeroed when `zero`) buffer of `bytes`, retiring the old one
  void regrow(DeviceBuffer& b, std::size_t bytes, bool zero) {
    DeviceBuffer fresh(bytes);
    if (zero) {
      flute_dev::dev_zero(fresh.p, fresh.bytes, nullptr);
      flute_dev::stream_sync(nullptr);
    }
    std::swap(b, fresh);
    if (fresh.p) retired.push_back(std::move(fresh));
  }

  void upload(const std::vector<std::uint8_t>& packed, const std::vector<std::uint16_t>& scales,
              const std::vector<std::uint32_t>& lut_words) {
    w = DeviceBuffer(packed.size());
    sc = DeviceBuffer(scales.size() * 2);
    lut = DeviceBuffer(lut_words.size() * 4);
    flute_dev::h2d(w.p, packed.data(), packed.size(), nullptr);
    flute_dev::h2d(sc.p, scales.data(), scales.size() * 2, nullptr);
    flute_dev::h2d(lut.p, lut_words.data(), lut_words.size() * 4, nullptr);
    // every m <= 32 default-worker call fits without growing (growth is a
    // synchronous allocation, not allowed inside CUDA-graph capture)
    reserve(32);
  }

  // Size the workspace for every call with m <= max_m and default workers.
  void reserve(int max_m) {
    std::size_t need = 0;
    for (int m = 1; m <= max_m; m = m < 32 ? std::min(32, m * 2) : m + 32)
      need = std::max(need, flute_dev::call_workspace_bytes(m, k, n, 0));
    need = std::max(need, flute_dev::call_workspace_bytes(max_m, k, n, 0));
    if (need > ws.bytes) regrow(ws, need, true);
    for (int m = 64; m <= max_m; m = m < 512 ? m * 2 : m + 512) grow_tc(m);
    grow_tc(max_m);
  }

  // the tcgen05 path's split-K partials: a buffer of their own, so the
  // Stream-K slots in `ws` are never touched by M >= 64 calls
  void grow_tc(int m) {
    const std::size_t need = flute_dev::tc_call_part_bytes(m, k, n);
    if (need > ws_tc.bytes) regrow(ws_tc, need, false);
  }

  // autotuned decomposition per m-class (row block 8 / 16 / 32), -1 = none
  flute_dev::Decomp tuned[3] = {};

  static int mclass(int m) { return m <= 8 ? 0 : m <= 16 ? 1 : m <= 32 ? 2 : -1; }

  // grow the workspace for an (m, workers) call (a synchronous allocation:
  // never inside CUDA-graph capture)
  void ensure_ws(int m, int workers) {
    const std::size_t need = flute_dev::call_workspace_bytes(m, k, n, workers);
    if (need > ws.bytes) regrow(ws, need, true);
    grow_tc(m);
  }

  void gemm(const void* x, int m, void* y, int workers, void* stream,
            void* const* y_peers = nullptr, int n_peers = 0, int ldy = 0, int ycol0 = 0,
            const flute_dev::Decomp* force = nullptr) {
    ensure_ws(m, workers);
    flute_dev::GemmArgs a;
    a.x = x;
    a.m = m;
    a.k = k;
    a.n = n;
    a.w = w.p;
    a.scales = sc.p;
    a.vlut = lut.p;
    a.bits = bits;
    a.group = group;
    a.y = y;
    a.workspace = ws.p;
    a.workspace_bytes = ws.bytes;
    a.tc_part = ws_tc.p;
    a.tc_part_bytes = ws_tc.bytes;
    a.workers = workers;
    a.stream = stream;
    a.y_peers = y_peers;
    a.n_peers = n_peers;
    a.ldy = ldy;
    a.ycol0 = ycol0;
    const int mc = mclass(m);
    const flute_dev::Decomp* d = force ? force : (workers <= 0 && mc >= 0 ? &tuned[mc] : nullptr);
    if (d && d->cluster >= 0) {
      a.cluster = d->cluster;
      a.workers = d->cluster == 0 ? d->workers : 0;
    }
    flute_dev::qgemm(a);
  }
};

DeviceWeights::DeviceWeights(const PackedWeights& pw, const std::vector<Half>& scales,
                             const VectorizedTable& lut, const QuantConfig& cfg)
    : impl_(std::make_unique<Impl>()) {
  cfg.validate(pw.k);
  if (pw.bits != cfg.bits || lut.bits != cfg.bits) {
    throw ConfigError("device weights: bit width mismatch between config, weights, and table");
  }
  impl_->k = pw.k;
  impl_->n = pw.n;
  impl_->bits = pw.bits;
  impl_->group = cfg.group_size;
  impl_->upload(pack_device_from_canonical(pw, cfg.group_size),
                scales_to_device(scales, pw.k, pw.n, cfg.group_size), device_vlut_words(lut));
}

DeviceWeights::DeviceWeights(const std::vector<std::uint8_t>& indices,
                             const std::vector<Half>& scales, const LookupTable& table, int k,
                             int n, const QuantConfig& cfg)
    : impl_(std::make_unique<Impl>()) {
  cfg.validate(k);
  if (table.bits != cfg.bits) throw ConfigError("device weights: table bit width mismatch");
  impl_->k = k;
  impl_->n = n;
  impl_->bits = cfg.bits;
  impl_->group = cfg.group_size;
  impl_->upload(pack_device(indices, k, n, cfg.bits, cfg.group_size),
                scales_to_device(scales, k, n, cfg.group_size),
                device_vlut_words(make_vectorized_lut(table, 1)));
}

DeviceWeights::DeviceWeights() : impl_(std::make_unique<Impl>()) {}

std::unique_ptr<DeviceWeights> DeviceWeights::from_device_indices(
    const std::uint8_t* idx_dev, const std::uint16_t* scales_dev, const std::vector<Half>& table16,
    int k, int n, const QuantConfig& cfg, void* stream) {
  cfg.validate(k);
  if (idx_dev == nullptr || scales_dev == nullptr) throw InputError("null device indices/scales");
  if (table16.size() != (std::size_t{1} << cfg.bits)) throw ConfigError("table size != 2^bits");
  const DeviceGeometry g = device_geometry(k, n, cfg.bits, cfg.group_size);
  std::unique_ptr<DeviceWeights> dw(new DeviceWeights());
  Impl& im = *dw->impl_;
  im.k = k;
  im.n = n;
  im.bits = cfg.bits;
  im.group = cfg.group_size;
  im.w = DeviceBuffer(g.weight_bytes());
  im.sc = DeviceBuffer(g.scale_bytes());
  flute_dev::pack_device_on_device(idx_dev, k, n, cfg.bits, cfg.group_size,
                                   static_cast<std::uint8_t*>(im.w.p), stream);
  flute_dev::scales_device_on_device(scales_dev, k, n, cfg.group_size,
                                     static_cast<std::uint16_t*>(im.sc.p), stream);
  LookupTable t;
  t.bits = cfg.bits;
  for (const Half h : table16) t.values.push_back(f16_to_f32(h));
  const std::vector<std::uint32_t> words = device_vlut_words(make_vectorized_lut(t, 1));
  im.lut = DeviceBuffer(words.size() * 4);
  flute_dev::h2d(im.lut.p, words.data(), words.size() * 4, stream);
  flute_dev::stream_sync(stream);
  im.reserve(32);
  return dw;
}

std::unique_ptr<DeviceWeights> DeviceWeights::from_flte(const FlteModel& model, void* stream) {
  const int k = model.k, n = model.n, bits = model.cfg.bits;
  const std::size_t words0 = model.slices.at(0).words.size();
  const std::size_t words1 = bits == 3 ? model.slices.at(1).words.size() : 0;
  DeviceBuffer s0(words0 * 4), s1(words1 * 4 + 4), idx(static_cast<std::size_t>(k) * n),
      sc(model.scales.size() * 2);
  flute_dev::h2d(s0.p, model.slices[0].words.data(), words0 * 4, stream);
  if (bits == 3) flute_dev::h2d(s1.p, model.slices[1].words.data(), words1 * 4, stream);
  flute_dev::h2d(sc.p, model.scales.data(), model.scales.size() * 2, stream);
  const LayoutDescriptor& L = model.layout;
  const int lay[6] = {L.tile_m, L.tile_n, L.tile_k, L.frag_m, L.frag_n, L.frag_k};
  flute_dev::unpack_canonical_device(static_cast<const std::uint32_t*>(s0.p),
                                     static_cast<const std::uint32_t*>(s1.p), k, n, bits, lay,
                                     static_cast<std::uint8_t*>(idx.p), stream);
  auto dw = from_device_indices(static_cast<const std::uint8_t*>(idx.p),
                                static_cast<const std::uint16_t*>(sc.p), model.table, k, n,
                                model.cfg, stream);
  return dw;  // (from_device_indices synchronised the stream before the temporaries go)
}

void quantize_on_device(const float* w_dev, int k, int n, const QuantConfig& cfg,
                        std::uint8_t* idx_dev, std::uint16_t* scales_dev, void* stream) {
  cfg.validate(k);
  if (n < 1) throw ConfigError("quantize: n must be positive");
  if (w_dev == nullptr || idx_dev == nullptr || scales_dev == nullptr)
    throw InputError("quantize: null device pointer");
  const LookupTable t = build_nf_table(cfg.bits);
  flute_dev::quantize_device(w_dev, k, n, cfg.bits, cfg.group_size, t.values.data(), idx_dev,
                             scales_dev, stream);
}

DeviceWeights::~DeviceWeights() = default;
int DeviceWeights::k() const { return impl_->k; }
void DeviceWeights::reserve(int max_m) { impl_->reserve(max_m); }

std::string DeviceWeights::autotune(int m, void* stream, int reps) {
  Impl& im = *impl_;
  const int mc = Impl::mclass(m);
  if (mc < 0) throw ConfigError("autotune: m must be in [1, 32] (the memory-bound kernel)");
  if (reps < 1) reps = 1;
  DeviceBuffer x(static_cast<std::size_t>(m) * im.k * 2), y(static_cast<std::size_t>(m) * im.n * 2);
  flute_dev::dev_zero(x.p, x.bytes, stream);
  const std::vector<flute_dev::Decomp> cands = flute_dev::decomp_candidates(m, im.k, im.n, im.bits);
  for (const flute_dev::Decomp& c : cands) {  // grow the workspace before timing
    if (c.cluster == 0) {
      const std::size_t need = flute_dev::workspace_bytes(m, c.workers);
      if (need > im.ws.bytes) im.regrow(im.ws, need, true);
    }
  }
  double best_t = 1e30;
  flute_dev::Decomp best{};
  std::string report;
  for (const flute_dev::Decomp& c : cands) {
    auto run = [&] { im.gemm(x.p, m, y.p, 0, stream, nullptr, 0, 0, 0, &c); };
    for (int i = 0; i < 3; ++i) run();
    const double t = flute_dev::time_launches(run, reps, stream);
    report += "cluster=" + std::to_string(c.cluster) + " workers=" + std::to_string(c.workers) +
              ": " + std::to_string(t) + " us\n";
    if (t < best_t) {
      best_t = t;
      best = c;
    }
  }
  im.tuned[mc] = best;
  return report;
}
int DeviceWeights::n() const { return impl_->n; }

void DeviceWeights::gemm(const Half* x_dev, int m, Half* y_dev, int workers, void* stream) {
  impl_->gemm(x_dev, m, y_dev, workers, stream);
}

void DeviceWeights::gemm_peers(const Half* x_dev, int m, void* const* y_peers, int n_peers,
                               int ldy, int ycol0, int workers, void* stream) {
  if (n_peers < 1) throw ConfigError("gemm_peers: need at least one output buffer");
  impl_->gemm(x_dev, m, nullptr, workers, stream, y_peers, n_peers, ldy, ycol0);
}

MatH DeviceWeights::gemm_host(const MatH& x, int workers, void* stream) {
  if (x.cols != impl_->k) throw ConfigError("gemm_host: activation K does not match weight K");
  MatH y(x.rows, impl_->n);
  gemm_host_raw(reinterpret_cast<const std::uint16_t*>(x.data.data()), x.rows,
                reinterpret_cast<std::uint16_t*>(y.data.data()), workers, stream);
  return y;
}

void DeviceWeights::gemm_host_raw(const std::uint16_t* x_host, int m, std::uint16_t* y_host,
                                  int workers, void* stream) {
  if (m < 1) throw ConfigError("gemm_host: m must be >= 1");
  const std::size_t xb = static_cast<std::size_t>(m) * impl_->k * 2;
  const std::size_t yb = static_cast<std::size_t>(m) * impl_->n * 2;
  if (impl_->xbuf.bytes < xb) impl_->regrow(impl_->xbuf, xb, false);
  if (impl_->ybuf.bytes < yb) impl_->regrow(impl_->ybuf, yb, false);
  flute_dev::h2d(impl_->xbuf.p, x_host, xb, stream);
  impl_->gemm(impl_->xbuf.p, m, impl_->ybuf.p, workers, stream);
  flute_dev::d2h(y_host, impl_->ybuf.p, yb, stream);
  flute_dev::stream_sync(stream);
}

std::vector<flute_dev::HostBatchItem> DeviceWeights::batch_items(
    DeviceWeights* const* ws, const std::uint16_t* const* x_host, const int* m,
    std::uint16_t* const* y_host, int count, int workers) {
  if (count < 0) throw ConfigError("gemm_host_batch: count must be >= 0");
  std::vector<flute_dev::HostBatchItem> items(static_cast<std::size_t>(count));
  for (int i = 0; i < count; ++i) {
    if (ws[i] == nullptr || x_host[i] == nullptr || y_host[i] == nullptr)
      throw InputError("gemm_host_batch: null handle or buffer at item " + std::to_string(i));
    if (m[i] < 1) throw ConfigError("gemm_host_batch: m must be >= 1");
    Impl* im = ws[i]->impl_.get();
    const int mi = m[i];
    items[i].gemm = [im, mi, workers](const void* x, void* y, void* st) {
      im->gemm(x, mi, y, workers, st);
    };
    items[i].prepare = [im, mi, workers]() { im->ensure_ws(mi, workers); };
    items[i].x_host = x_host[i];
    items[i].x_bytes = static_cast<std::size_t>(mi) * im->k * 2;
    items[i].y_host = y_host[i];
    items[i].y_bytes = static_cast<std::size_t>(mi) * im->n * 2;
  }
  return items;
}

void DeviceWeights::gemm_host_batch(DeviceWeights* const* ws, const std::uint16_t* const* x_host,
                                    const int* m, std::uint16_t* const* y_host, int count,
                                    int workers, void* stream) {
  flute_dev::host_batch(batch_items(ws, x_host, m, y_host, count, workers), stream);
}

HostBatch::HostBatch(DeviceWeights* const* ws, const std::uint16_t* const* x_host, const int* m,
                     std::uint16_t* const* y_host, int count, int workers)
    : graph_(flute_dev::host_batch_capture(
          DeviceWeights::batch_items(ws, x_host, m, y_host, count, workers))) {}

HostBatch::~HostBatch() { flute_dev::host_batch_free(graph_); }

void HostBatch::run(void* stream) { flute_dev::host_batch_run(graph_, stream); }

// ---------------------------------------------------------------------------
// Reference API
// ---------------------------------------------------------------------------

MatmulResult execute(const MatmulProblem& problem) {
  if (problem.x == nullptr || problem.weights == nullptr || problem.scales == nullptr ||
      problem.lut == nullptr) {
    throw InputError("matmul: problem is missing inputs");
  }
  const PackedWeights& pw = *problem.weights;
  if (problem.x->cols != pw.k) {
    throw ConfigError("matmul: activation K (" + std::to_string(problem.x->cols) +
                      ") does not match weight K (" + std::to_string(pw.k) + ")");
  }
  if (problem.cfg.bits != pw.bits || problem.lut->bits != pw.bits) {
    throw ConfigError("matmul: bit width mismatch between config, weights, and table");
  }
  const long expected = static_cast<long>(pw.k) * pw.n / problem.cfg.group_size;
  if (static_cast<long>(problem.scales->size()) != expected) {
    throw InputError("matmul: expected " + std::to_string(expected) + " scales, got " +
                     std::to_string(problem.scales->size()));
  }
  const Shape s = make_shape(problem.x->rows, pw.k, pw.n, pw.layout, problem.cfg, problem.tile_m,
                             problem.stages, problem.workers);
  DeviceWeights dw(pw, *problem.scales, *problem.lut, problem.cfg);
  MatmulResult r;
  r.y = dw.gemm_host(*problem.x, problem.workers, nullptr);
  r.stats = account(s, problem.workers);
  return r;
}

ShardRange shard_range(int k, int n, int bits, int group, int world, int rank) {
  if (world < 1 || rank < 0 || rank >= world) {
    throw ConfigError("shard_range: need world >= 1 and 0 <= rank < world");
  }
  const DeviceGeometry g = device_geometry(k, n, bits, group);
  const int T = g.tiles_n();
  if (world > T) throw ConfigError("shard_range: more ranks than 64-column tiles");
  const int t0 = static_cast<int>(static_cast<long>(T) * rank / world);
  const int t1 = static_cast<int>(static_cast<long>(T) * (rank + 1) / world);
  ShardRange r;
  r.n0 = t0 * kUnitN;
  r.n1 = std::min(t1 * kUnitN, n);
  const std::size_t tile_w = g.unit_bytes() * static_cast<std::size_t>(g.tiles_k());
  const std::size_t tile_s = static_cast<std::size_t>(g.groups_padded()) * kUnitN * 2;
  r.w_off = tile_w * t0;
  r.w_bytes = tile_w * (t1 - t0);
  r.s_off = tile_s * t0;
  r.s_bytes = tile_s * (t1 - t0);
  return r;
}

double bits_per_param(const QuantConfig& cfg) {
  cfg.validate();
  return cfg.bits + 16.0 / cfg.group_size;
}

double weight_traffic_ratio(const TrafficStats& stats, double dense_weight_bytes) {
  if (dense_weight_bytes <= 0.0) {
    throw InputError("weight_traffic_ratio: dense byte count must be positive");
  }
  return static_cast<double>(stats.bytes_weights + stats.bytes_scales) / dense_weight_bytes;
}

TrafficStats plan_traffic(const ProblemShape& shape) {
  const Shape s = make_shape(shape.m, shape.k, shape.n, shape.layout, shape.cfg, shape.tile_m,
                             shape.stages, shape.workers);
  return account(s, shape.workers);
}

void mma_fragment(std::span<const Half> a, std::span<const Half> b, std::span<float> c,
                  const FragDims& dims) {
  const auto m = static_cast<std::size_t>(dims.m), n = static_cast<std::size_t>(dims.n),
             k = static_cast<std::size_t>(dims.k);
  if (dims.m <= 0 || dims.n <= 0 || dims.k <= 0 || a.size() != m * k || b.size() != k * n ||
      c.size() != m * n) {
    throw ConfigError("mma_fragment: fragment shape mismatch (m=" + std::to_string(dims.m) +
                      " n=" + std::to_string(dims.n) + " k=" + std::to_string(dims.k) + ")");
  }
  flute_dev::mma_fragment(reinterpret_cast<const std::uint16_t*>(a.data()),
                          reinterpret_cast<const std::uint16_t*>(b.data()), c.data(), dims.m,
                          dims.n, dims.k);
}

}  // namespace flutesim
