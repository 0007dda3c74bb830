// flute-b200 — internal interface between the C++ host layer and the CUDA
// translation units.  No CUDA types: streams are void* (cudaStream_t).
// Every function throws flutesim::{ConfigError, InputError, CudaError}.
#pragma once

#include <cstddef>
#include <cstdint>
#include <functional>
#include <vector>

namespace flute_dev {

struct GemmArgs {
  const void* x = nullptr;       // f16 [m][k], device
  int m = 0, k = 0, n = 0;
  const void* w = nullptr;       // device-layout weights, device
  const void* scales = nullptr;  // device-layout scales, device
  const void* vlut = nullptr;    // 2^(2b) device-order u32 words, device
  int bits = 4, group = 128;
  void* y = nullptr;             // f16 [m][n], device
  // Fused all-gather (N-sharded layer): when n_peers > 0, Y is stored to every
  // y_peers[i] (device pointers reachable from this GPU: peer / multicast
  // mappings) at [row * ldy + ycol0 + col]; y is then ignored.
  void* const* y_peers = nullptr;
  int n_peers = 0;
  int ldy = 0, ycol0 = 0;
  void* workspace = nullptr;
  std::size_t workspace_bytes = 0;
  // Optional separate buffer for the tcgen05 path's split-K partials (M >= 64).
  // Without it the partials go to `workspace`, which the Stream-K path also
  // uses, and the reduce kernel must re-zero them (slower).
  void* tc_part = nullptr;
  std::size_t tc_part_bytes = 0;
  int workers = 0;               // <= 0: default
  void* stream = nullptr;
  // Decomposition override (autotuner): cluster >= 1 forces cluster split-K
  // with that cluster size (workers ignored); 0 = Stream-K with `workers`;
  // -1 = heuristic.
  int cluster = -1;
};

// Candidate decompositions for an m-row call (autotuner): {cluster, workers}.
struct Decomp {
  int cluster = -1, workers = 0;
};
std::vector<Decomp> decomp_candidates(int m, int k, int n, int bits);
// Mean device time (us) of `fn` (one launch sequence on `stream`), each rep
// preceded by an untimed write of a buffer larger than L2 so weights stream
// from HBM as in real use.
double time_launches(const std::function<void()>& fn, int reps, void* stream);

void qgemm(const GemmArgs& a);

// Compute-bound path (qgemm_tc.cu): tcgen05/TMEM kernel used by qgemm() for
// m >= 64 (unless FLUTE_NO_TC is set).  Split-K partials live in the caller's
// workspace; tc_workspace_bytes is the size for the full split count.
bool tc_enabled(int m);
std::size_t tc_workspace_bytes(int m, int k, int n, int sms);
// Split-K partial bytes of the tcgen05 path for an m-row call (0 if m < 64).
std::size_t tc_call_part_bytes(int m, int k, int n);
void qgemm_tc(const GemmArgs& a, int tiles_k, int tiles_n, int gp, int sms, bool zero_part, void* part,
              std::size_t part_bytes);
// Workspace a qgemm call with these dimensions needs (either path).
std::size_t call_workspace_bytes(int m, int k, int n, int workers);
std::size_t workspace_bytes(int m, int workers);
// co-resident CTA slots of the memory-bound kernel for an m-row call
int max_workers(int m, int bits = 3);
int default_workers(int m, int k, int n, int bits);
int sm_count(int device);
int device_count();

// FLUTE_DEBUG_TIMES=1 per-CTA timeline of the last qgemm launch (8 u64 / CTA).
void debug_times(unsigned long long* out, int workers);

// Device self-checks.
void dequant_all(const std::uint32_t* vlut_dev_words_host, int bits, const std::uint16_t* scales,
                 int n_scales, std::uint32_t* out_host);
void mma_fragment(const std::uint16_t* a, const std::uint16_t* b, float* c, int m, int n, int k);

// Weight preparation on the device (prep_kernels.cu).
void quantize_device(const float* w, int k, int n, int bits, int group, const float* table_host,
                     std::uint8_t* idx, std::uint16_t* scales, void* stream);
void unpack_canonical_device(const std::uint32_t* s0, const std::uint32_t* s1, int k, int n,
                             int bits, const int* layout6, std::uint8_t* idx, void* stream);
void pack_device_on_device(const std::uint8_t* idx, int k, int n, int bits, int group,
                           std::uint8_t* out, void* stream);
void scales_device_on_device(const std::uint16_t* sc, int k, int n, int group,
                             std::uint16_t* out, void* stream);

// Learned-sigma refinement state (refine_kernels.cu): W f32 [k][n] and X f32
// [m][k] uploaded once; evaluate() runs one straight-through evaluation at the
// device sigma and returns the loss; descend() applies sigma -= lr * grad.
class SteDevice {
 public:
  SteDevice(const float* w_host, const float* x_host, int m, int k, int n, int group,
            const std::vector<double>& quantiles);
  ~SteDevice();
  SteDevice(const SteDevice&) = delete;
  SteDevice& operator=(const SteDevice&) = delete;
  void set_sigma(const double* sigma_host);
  double evaluate();
  void descend(double lr);
  // any pointer may be null
  void get(double* sigma, double* grad, std::uint8_t* idx, float* absmax) const;
  long groups() const { return groups_; }

 private:
  int m_, k_, n_, group_, nq_;
  long groups_ = 0;
  float* w_ = nullptr;
  float* x_ = nullptr;
  double* q_ = nullptr;
  double* sigma_ = nullptr;
  double* grad_ = nullptr;
  float* absmax_ = nullptr;
  std::uint8_t* idx_ = nullptr;
  double* d_ = nullptr;
  double* e_ = nullptr;
  double* scalars_ = nullptr;
  unsigned long long* bad_ = nullptr;
};

// A batch of GEMMs on host buffers (host_batch, qgemm_mma.cu): H2D of every
// input on an internal copy stream, item i's GEMM on `stream` once its input
// has landed, D2H of its output on a second copy stream; returns when every
// output is in host memory.  gemm(x_dev, y_dev, stream) enqueues one GEMM.
struct HostBatchItem {
  std::function<void(const void*, void*, void*)> gemm;
  std::function<void()> prepare;  // size the handle's workspace (before capture)
  const void* x_host = nullptr;
  std::size_t x_bytes = 0;
  void* y_host = nullptr;
  std::size_t y_bytes = 0;
};
void host_batch(const std::vector<HostBatchItem>& items, void* stream);
// The same batch captured once into a CUDA graph (own staging buffers and
// copy streams); run replays it on `stream` and synchronises.
struct HostBatchGraph;
HostBatchGraph* host_batch_capture(const std::vector<HostBatchItem>& items);
void host_batch_run(HostBatchGraph* g, void* stream);
void host_batch_free(HostBatchGraph* g);

// N-sharded layer (shard_kernels.cu): shard-major [P][m][w_max] all-gather
// result -> row-major Y [m][n] (n0s_dev: P + 1 column starts, device); and the
// release/acquire flag barrier of the fused path (flags[r]: rank r's [2][P]
// flag array as mapped on this GPU).
void shard_relayout(const void* gathered, void* y, int m, int n, int world, int w_max, const int* n0s_dev,
                    void* stream);
void peer_barrier(std::uint32_t* const* flags, int world, int me, int b, std::uint32_t epoch, void* stream);

// Small RAII device buffer helpers used by the host layer.
void* dev_alloc(std::size_t bytes);
void dev_free(void* p);
void h2d(void* dst, const void* src, std::size_t bytes, void* stream);
void d2h(void* dst, const void* src, std::size_t bytes, void* stream);
void dev_zero(void* p, std::size_t bytes, void* stream);
void stream_sync(void* stream);

}  // namespace flute_dev
