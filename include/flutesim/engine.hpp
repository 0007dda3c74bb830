// flute-b200 — the fused LUT-dequant matmul ("qgemm").
//
// Drop-in for the reference engine (reference: proj/include/flutesim/
// engine.hpp:24-96, engine.cpp:345-418).  execute() keeps the reference's
// signature, validation and exception classes, but the work runs on the B200:
// the packed weights are re-laid into sm_100a fragment order, uploaded, and one
// Stream-K kernel does TMA-fed dequant + tensor-core MMA with a deterministic
// fp32 cross-CTA fixup.  Results are bitwise identical across runs, ExecMode
// and `stages`; `workers` is the Stream-K CTA count.
//
// TrafficStats keeps the reference's *accounting model* (engine.cpp:87-130):
// execute().stats == plan_traffic(shape) exactly, as the reference guarantees.
// It is not a measurement of the GPU kernel (use ncu / bench.py for that).
#pragma once

#include <cstdint>
#include <memory>
#include <vector>
#include <string>

#include "flutesim/matrix.hpp"
#include "flutesim/pack.hpp"
#include "flutesim/quantize.hpp"
#include "flutesim/streamk.hpp"
#include "flutesim/vec_lut.hpp"

namespace flute_dev {
struct HostBatchItem;
struct HostBatchGraph;
}  // namespace flute_dev

namespace flutesim {

struct TrafficStats {
  std::uint64_t bytes_weights = 0;
  std::uint64_t bytes_scales = 0;
  std::uint64_t bytes_table = 0;
  std::uint64_t bytes_activations = 0;
  std::uint64_t bytes_partials_rw = 0;
  std::uint64_t bytes_output = 0;
  std::uint64_t flops = 0;

  std::uint64_t total_bytes() const {
    return bytes_weights + bytes_scales + bytes_table + bytes_activations + bytes_partials_rw +
           bytes_output;
  }
  double arithmetic_intensity() const {
    return total_bytes() == 0 ? 0.0
                              : static_cast<double>(flops) / static_cast<double>(total_bytes());
  }
  TrafficStats& operator+=(const TrafficStats& o);
};

enum class ExecMode {
  kSerial,    // accepted for API compatibility; same GPU kernel, same bits
  kParallel,
};

struct MatmulProblem {
  const MatH* x = nullptr;
  const PackedWeights* weights = nullptr;
  const std::vector<Half>* scales = nullptr;
  const VectorizedTable* lut = nullptr;
  QuantConfig cfg;
  int workers = 1;   // Stream-K CTAs on the device
  int stages = 2;    // validated (>= 1); the device pipeline depth is its own
  int tile_m = 0;
  ExecMode mode = ExecMode::kParallel;
};

struct MatmulResult {
  MatH y;
  TrafficStats stats;
};

MatmulResult execute(const MatmulProblem& problem);

// quantize_matrix (quantize.hpp:45) on the GPU for a device-resident f32
// [k][n] matrix: indices [k][n] and binary16 scales [n][k/g] into device
// buffers, bit-exact with the host quantizer (synchronises `stream`; throws
// InputError on non-finite weights or binary16 overflow).
void quantize_on_device(const float* w_dev, int k, int n, const QuantConfig& cfg,
                        std::uint8_t* idx_dev, std::uint16_t* scales_dev, void* stream = nullptr);

double bits_per_param(const QuantConfig& cfg);
double weight_traffic_ratio(const TrafficStats& stats, double dense_weight_bytes);

struct ProblemShape {
  int m = 1;
  int k = 0;
  int n = 0;
  QuantConfig cfg;
  LayoutDescriptor layout;
  int workers = 1;
  int stages = 2;
  int dup = 1;
  int tile_m = 0;
};
TrafficStats plan_traffic(const ProblemShape& shape);

// ---------------------------------------------------------------------------
// N-column sharding: rank r of `world` owns the 64-column
// tiles [r*T/world, (r+1)*T/world) of the T = ceil(n/64) tiles, i.e. columns
// [n0, n1).  Because device-layout units are n-tile major, the shard's packed
// weights and scales are one contiguous byte range of the full device buffers.
// ---------------------------------------------------------------------------

struct ShardRange {
  int n0 = 0, n1 = 0;                  // columns
  std::size_t w_off = 0, w_bytes = 0;  // into the full device-layout weights
  std::size_t s_off = 0, s_bytes = 0;  // into the full device-layout scales
};
ShardRange shard_range(int k, int n, int bits, int group, int world, int rank);

// ---------------------------------------------------------------------------
// Device-resident path (new): upload once, call many times.
// ---------------------------------------------------------------------------

class DeviceWeights {
 public:
  // From the canonical packed form + scales + vLUT (what execute() receives).
  DeviceWeights(const PackedWeights& pw, const std::vector<Half>& scales,
                const VectorizedTable& lut, const QuantConfig& cfg);
  // From a raw index matrix [k][n] + [n][k/g] scales + table values.
  DeviceWeights(const std::vector<std::uint8_t>& indices, const std::vector<Half>& scales,
                const LookupTable& table, int k, int n, const QuantConfig& cfg);
  // From device-resident indices [k][n] u8 + scales [n][k/g] (binary16 bits),
  // e.g. straight out of quantize_on_device: packed into the device layout on
  // the GPU.  `table16` are the 2^bits binary16 table values.
  static std::unique_ptr<DeviceWeights> from_device_indices(const std::uint8_t* idx_dev,
                                                            const std::uint16_t* scales_dev,
                                                            const std::vector<Half>& table16, int k,
                                                            int n, const QuantConfig& cfg,
                                                            void* stream = nullptr);
  // From an FLTE container (flte.hpp): the canonical slices are uploaded as
  // stored and re-permuted to the device layout on the GPU.
  static std::unique_ptr<DeviceWeights> from_flte(const struct FlteModel& model,
                                                  void* stream = nullptr);
  ~DeviceWeights();
  DeviceWeights(const DeviceWeights&) = delete;
  DeviceWeights& operator=(const DeviceWeights&) = delete;

  int k() const;
  int n() const;
  // Pre-size the device workspace for calls with m <= max_m (default workers),
  // so no later call allocates (e.g. inside CUDA-graph capture).  Calls with
  // m <= 32 never allocate; larger m (tcgen05 split-K partials) may on first use.
  void reserve(int max_m);
  // Time the candidate decompositions (cluster split-K sizes, Stream-K worker
  // counts) for m-row calls on this weight shape and keep the fastest for
  // later default-worker calls of the same row class (M <= 8 / 16 / 32);
  // returns the timing report.  The paper's "compile several instantiations,
  // keep the best", at run time.
  std::string autotune(int m, void* stream = nullptr, int reps = 20);
  // y_dev[m][n] = x_dev[m][k] * W_hat, device pointers, async on `stream`.
  void gemm(const Half* x_dev, int m, Half* y_dev, int workers = 0, void* stream = nullptr);
  // N-sharded layer: store this GEMM's [m][n] result into every y_peers[i]
  // (device pointers reachable from this GPU — NVLink peer or multicast
  // mappings) at [row * ldy + ycol0 + col]: the all-gather fused into the
  // epilogue.  The caller synchronises ranks before reading the full Y.
  void gemm_peers(const Half* x_dev, int m, void* const* y_peers, int n_peers, int ldy, int ycol0,
                  int workers = 0, void* stream = nullptr);
  // Host in / host out (copies inside; synchronizes the stream).
  MatH gemm_host(const MatH& x, int workers = 0, void* stream = nullptr);
  // Raw host buffers (f16 bits; pinned memory makes the copies truly async).
  void gemm_host_raw(const std::uint16_t* x_host, int m, std::uint16_t* y_host, int workers = 0,
                     void* stream = nullptr);
  // A batch of GEMMs on host buffers (one per handle; a handle may repeat):
  // input copies, GEMMs and output copies pipelined across three streams
  // (GEMMs on `stream`); returns when every y_host[i] holds its result.
  static void gemm_host_batch(DeviceWeights* const* ws, const std::uint16_t* const* x_host,
                              const int* m, std::uint16_t* const* y_host, int count,
                              int workers = 0, void* stream = nullptr);
  // (internal) the per-item closures behind gemm_host_batch / HostBatch
  static std::vector<flute_dev::HostBatchItem> batch_items(DeviceWeights* const* ws,
                                                           const std::uint16_t* const* x_host,
                                                           const int* m,
                                                           std::uint16_t* const* y_host, int count,
                                                           int workers);

  struct Impl;

 private:
  DeviceWeights();
  std::unique_ptr<Impl> impl_;
};

// A gemm_host_batch prepared once and captured as a CUDA graph: input copies
// (from the given host buffers), the GEMMs and the output copies, with their
// cross-stream dependencies.  run() replays it on `stream` and returns when
// every output is on the host.  The handles and host buffers must outlive it;
// refill the host inputs in place between runs.
class HostBatch {
 public:
  HostBatch(DeviceWeights* const* ws, const std::uint16_t* const* x_host, const int* m,
            std::uint16_t* const* y_host, int count, int workers = 0);
  ~HostBatch();
  HostBatch(const HostBatch&) = delete;
  HostBatch& operator=(const HostBatch&) = delete;
  void run(void* stream = nullptr);

 private:
  flute_dev::HostBatchGraph* graph_;
};

}  // namespace flutesim
