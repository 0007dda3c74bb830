// flute-b200 — host side of the N-column-sharded layer (include/flutesim/
// sharded.hpp).
//
// Communicator: NCCL loaded at run time through dlopen/dlsym (no link-time
// dependency: inside a PyTorch process the already-loaded libnccl.so.2 is
// reused, so one NCCL serves both).  ShardedWeights: the rank's column slice
// uploaded as an ordinary DeviceWeights, plus
//  * the NCCL path: a [m][w] slice buffer, ncclAllGather into a shard-major
//    [P][m][w] buffer (straight into Y when m = 1 and the slices are equal),
//    and a re-layout kernel;
//  * the fused path: a double-buffered [2][max_m][n] output arena + a [2][P]
//    flag array per rank, exchanged once as CUDA IPC handles over NCCL; the
//    GEMM epilogue stores into every rank's arena (flute_dev::qgemm with peer
//    outputs) and a one-block kernel runs the release/acquire flag barrier.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <string>

#include "device_api.h"
#include "flutesim/errors.hpp"
#include "flutesim/sharded.hpp"

namespace flutesim {

namespace {

void cuda_ok(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

// The handful of NCCL entry points the layer needs.
struct Nccl {
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;

  void check(ncclResult_t r, const char* what) const {
    if (r != ncclSuccess) {
      throw CudaError(std::string(what) + ": " + (error_string ? error_string(r) : "NCCL error") + " (" +
                      std::to_string(static_cast<int>(r)) + ")");
    }
  }
};

const Nccl& nccl() {
  static Nccl api;
  static std::once_flag once;
  static std::string err;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_LOCAL);
    if (!h) {
      err = std::string("libnccl.so.2 not found: ") + dlerror();
      return;
    }
    auto sym = [&](const char* name) {
      void* p = dlsym(h, name);
      if (!p && err.empty()) err = std::string("NCCL symbol missing: ") + name;
      return p;
    };
    api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(sym("ncclGetUniqueId"));
    api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(sym("ncclCommInitRank"));
    api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(sym("ncclCommDestroy"));
    api.all_gather = reinterpret_cast<decltype(api.all_gather)>(sym("ncclAllGather"));
    api.error_string = reinterpret_cast<decltype(api.error_string)>(sym("ncclGetErrorString"));
  });
  if (!err.empty()) throw CudaError(err);
  return api;
}

}  // namespace

// ---------------------------------------------------------------------------
// Communicator
// ---------------------------------------------------------------------------

std::vector<std::uint8_t> Communicator::unique_id() {
  static_assert(sizeof(ncclUniqueId) == kIdBytes, "NCCL unique id size");
  ncclUniqueId id;
  nccl().check(nccl().get_unique_id(&id), "ncclGetUniqueId");
  std::vector<std::uint8_t> out(kIdBytes);
  std::memcpy(out.data(), &id, kIdBytes);
  return out;
}

Communicator::Communicator(const std::uint8_t* id, int world, int rank) : world_(world), rank_(rank) {
  if (id == nullptr) throw InputError("communicator: null unique id");
  if (world < 1 || world > 8 || rank < 0 || rank >= world)
    throw ConfigError("communicator: need 1 <= world <= 8 (one node) and 0 <= rank < world");
  ncclUniqueId uid;
  std::memcpy(&uid, id, kIdBytes);
  ncclComm_t c = nullptr;
  nccl().check(nccl().comm_init_rank(&c, world, uid, rank), "ncclCommInitRank");
  comm_ = c;
}

Communicator::~Communicator() {
  if (comm_) nccl().comm_destroy(static_cast<ncclComm_t>(comm_));
}

void Communicator::all_gather(const void* send_dev, void* recv_dev, std::size_t bytes, void* stream) {
  nccl().check(nccl().all_gather(send_dev, recv_dev, bytes, ncclUint8, static_cast<ncclComm_t>(comm_),
                                 static_cast<cudaStream_t>(stream)),
               "ncclAllGather");
}

// ---------------------------------------------------------------------------
// ShardedWeights
// ---------------------------------------------------------------------------

struct ShardedWeights::Impl {
  Communicator* comm = nullptr;
  int k = 0, n = 0, world = 1, rank = 0, max_m = 0;
  std::vector<ShardRange> ranges;
  int w_max = 0;
  bool equal = true;
  std::unique_ptr<DeviceWeights> local;
  // NCCL path
  void* slice = nullptr;     // [m][w_max]
  void* gathered = nullptr;  // [P][m][w_max]
  int cap_m = 0;             // rows the two buffers above hold
  int* n0s_dev = nullptr;    // [P + 1] column starts
  // fused path
  void* arena = nullptr;  // [2][max_m][n] f16, then [2][P] u32 flags (this rank's)
  std::size_t flag_off = 0;
  std::vector<void*> peer_arena;  // every rank's arena mapped here (self = arena)
  std::uint64_t calls = 0;

  ~Impl() {
    for (int r = 0; r < static_cast<int>(peer_arena.size()); ++r)
      if (r != rank && peer_arena[r]) cudaIpcCloseMemHandle(peer_arena[r]);
    flute_dev::dev_free(arena);
    flute_dev::dev_free(slice);
    flute_dev::dev_free(gathered);
    flute_dev::dev_free(n0s_dev);
  }

  void grow(int m) {
    if (m <= cap_m) return;
    flute_dev::dev_free(slice);
    flute_dev::dev_free(gathered);
    slice = gathered = nullptr;
    slice = flute_dev::dev_alloc(static_cast<std::size_t>(m) * w_max * 2);
    gathered = flute_dev::dev_alloc(static_cast<std::size_t>(world) * m * w_max * 2);
    cap_m = m;
  }

  // One-time: the output arena + flags, exchanged as IPC handles over NCCL.
  void setup_peers() {
    const std::size_t ybytes = 2 * static_cast<std::size_t>(max_m) * n * 2;
    flag_off = (ybytes + 255) / 256 * 256;
    const std::size_t total = flag_off + 2 * static_cast<std::size_t>(world) * 4;
    arena = flute_dev::dev_alloc(total);
    cuda_ok(cudaMemset(arena, 0, total), "arena clear");
    peer_arena.assign(world, nullptr);
    peer_arena[rank] = arena;
    if (world == 1) return;
    cudaIpcMemHandle_t mine;
    cuda_ok(cudaIpcGetMemHandle(&mine, arena), "cudaIpcGetMemHandle");
    void* d_send = flute_dev::dev_alloc(sizeof(mine));
    void* d_recv = flute_dev::dev_alloc(sizeof(mine) * world);
    cudaStream_t st = nullptr;
    try {
      cuda_ok(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "stream");
      cuda_ok(cudaMemcpyAsync(d_send, &mine, sizeof(mine), cudaMemcpyHostToDevice, st), "h2d");
      comm->all_gather(d_send, d_recv, sizeof(mine), st);
      std::vector<cudaIpcMemHandle_t> all(world);
      cuda_ok(cudaMemcpyAsync(all.data(), d_recv, sizeof(mine) * world, cudaMemcpyDeviceToHost, st), "d2h");
      cuda_ok(cudaStreamSynchronize(st), "sync");
      for (int r = 0; r < world; ++r) {
        if (r == rank) continue;
        cuda_ok(cudaIpcOpenMemHandle(&peer_arena[r], all[r], cudaIpcMemLazyEnablePeerAccess),
                "cudaIpcOpenMemHandle");
      }
    } catch (...) {
      if (st) cudaStreamDestroy(st);
      flute_dev::dev_free(d_send);
      flute_dev::dev_free(d_recv);
      throw;
    }
    cudaStreamDestroy(st);
    flute_dev::dev_free(d_send);
    flute_dev::dev_free(d_recv);
  }
};

ShardedWeights::ShardedWeights(Communicator& comm, const std::vector<std::uint8_t>& indices,
                               const std::vector<Half>& scales, const LookupTable& table, int k, int n,
                               const QuantConfig& cfg, int max_m)
    : impl_(std::make_unique<Impl>()) {
  cfg.validate(k);
  if (indices.size() != static_cast<std::size_t>(k) * n) throw InputError("sharded: indices must be k*n");
  if (scales.size() != static_cast<std::size_t>(n) * (k / cfg.group_size))
    throw InputError("sharded: scales must be n*k/group");
  if (max_m < 1) throw ConfigError("sharded: max_m must be >= 1");
  Impl& im = *impl_;
  im.comm = &comm;
  im.k = k;
  im.n = n;
  im.world = comm.world();
  im.rank = comm.rank();
  im.max_m = max_m;
  for (int r = 0; r < im.world; ++r) im.ranges.push_back(shard_range(k, n, cfg.bits, cfg.group_size, im.world, r));
  for (const ShardRange& r : im.ranges) {
    im.w_max = std::max(im.w_max, r.n1 - r.n0);
    im.equal = im.equal && (r.n1 - r.n0) == (im.ranges[0].n1 - im.ranges[0].n0);
  }
  const ShardRange& me = im.ranges[im.rank];
  const int w = me.n1 - me.n0;
  // the shard's columns of the index matrix and its rows of the [n][k/g] scales
  std::vector<std::uint8_t> idx(static_cast<std::size_t>(k) * w);
  for (int i = 0; i < k; ++i)
    std::memcpy(idx.data() + static_cast<std::size_t>(i) * w, indices.data() + static_cast<std::size_t>(i) * n + me.n0, w);
  const std::size_t gpc = static_cast<std::size_t>(k / cfg.group_size);
  std::vector<Half> sc(scales.begin() + static_cast<std::ptrdiff_t>(me.n0 * gpc),
                       scales.begin() + static_cast<std::ptrdiff_t>(me.n1 * gpc));
  im.local = std::make_unique<DeviceWeights>(idx, sc, table, k, w, cfg);
  im.local->reserve(max_m);
  std::vector<int> n0s(im.world + 1);
  for (int r = 0; r < im.world; ++r) n0s[r] = im.ranges[r].n0;
  n0s[im.world] = n;
  im.n0s_dev = static_cast<int*>(flute_dev::dev_alloc(n0s.size() * sizeof(int)));
  cuda_ok(cudaMemcpy(im.n0s_dev, n0s.data(), n0s.size() * sizeof(int), cudaMemcpyHostToDevice), "n0s");
  im.setup_peers();
}

ShardedWeights::~ShardedWeights() = default;

int ShardedWeights::n0() const { return impl_->ranges[impl_->rank].n0; }
int ShardedWeights::n1() const { return impl_->ranges[impl_->rank].n1; }
DeviceWeights& ShardedWeights::local() { return *impl_->local; }

void ShardedWeights::gemm(const Half* x_dev, int m, Half* y_dev, void* stream) {
  Impl& im = *impl_;
  if (m < 1) throw ConfigError("sharded gemm: m must be >= 1");
  if (x_dev == nullptr || y_dev == nullptr) throw InputError("sharded gemm: null device pointer");
  const ShardRange& me = im.ranges[im.rank];
  const int w = me.n1 - me.n0;
  im.grow(m);
  const std::size_t slice_bytes = static_cast<std::size_t>(m) * im.w_max * 2;
  if (w < im.w_max) flute_dev::dev_zero(im.slice, slice_bytes, stream);  // uneven: padded slice
  // the shard GEMM writes rows of w columns; the slice's row stride is w_max
  if (w == im.w_max) {
    im.local->gemm(x_dev, m, static_cast<Half*>(im.slice), 0, stream);
  } else {
    void* dst = im.slice;
    im.local->gemm_peers(x_dev, m, &dst, 1, im.w_max, 0, 0, stream);
  }
  if (m == 1 && im.equal) {
    // shard-major [P][1][w] == row-major [1][n]: gather straight into Y
    im.comm->all_gather(im.slice, y_dev, slice_bytes, stream);
    return;
  }
  im.comm->all_gather(im.slice, im.gathered, slice_bytes, stream);
  flute_dev::shard_relayout(im.gathered, y_dev, m, im.n, im.world, im.w_max, im.n0s_dev, stream);
}

const Half* ShardedWeights::gemm_fused(const Half* x_dev, int m, void* stream) {
  Impl& im = *impl_;
  if (m < 1 || m > im.max_m) throw ConfigError("sharded gemm_fused: need 1 <= m <= max_m");
  if (x_dev == nullptr) throw InputError("sharded gemm_fused: null x");
  const int b = static_cast<int>(im.calls & 1u);
  const std::uint32_t epoch = static_cast<std::uint32_t>(im.calls >> 1) + 1u;
  ++im.calls;
  const std::size_t ybuf = static_cast<std::size_t>(im.max_m) * im.n * 2;
  std::vector<void*> outs(im.world);
  std::vector<std::uint32_t*> flags(im.world);
  for (int r = 0; r < im.world; ++r) {
    outs[r] = static_cast<std::uint8_t*>(im.peer_arena[r]) + b * ybuf;
    flags[r] = reinterpret_cast<std::uint32_t*>(static_cast<std::uint8_t*>(im.peer_arena[r]) + im.flag_off);
  }
  im.local->gemm_peers(x_dev, m, outs.data(), im.world, im.n, n0(), 0, stream);
  flute_dev::peer_barrier(flags.data(), im.world, im.rank, b, epoch, stream);
  return reinterpret_cast<const Half*>(static_cast<const std::uint8_t*>(im.arena) + b * ybuf);
}

}  // namespace flutesim
