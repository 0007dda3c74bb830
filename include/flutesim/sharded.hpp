// flute-b200 — the N-column-sharded LUT-quantized layer over the GPUs of one
// node (BASELINE.json configs[3]: LLaMA-3-70B K=8192,
// N=28672 on 1/2/4/8 GPUs).  C++ host side of paper_2407_10960_b200/sharded.py.
//
// There is no reference counterpart (the reference is single-process CPU
// code); the shard of rank r is the reference's own GEMM (engine.cpp:345) on
// the column slice [n0, n1) of W, so every rank's Y columns equal the
// unsharded product's bitwise, and the only exchange is the output
// all-gather.
#pragma once

#include <cstdint>
#include <memory>
#include <vector>

#include "flutesim/engine.hpp"

namespace flutesim {

// One NCCL communicator over `world` ranks, one GPU per rank (the calling
// thread's current device).  NCCL is loaded at run time (libnccl.so.2: the
// copy already in the process — e.g. PyTorch's — else the system one).
class Communicator {
 public:
  static constexpr int kIdBytes = 128;
  // Rank 0 creates the id and distributes it out of band (e.g. a
  // torch.distributed broadcast or a file).
  static std::vector<std::uint8_t> unique_id();
  Communicator(const std::uint8_t* id, int world, int rank);
  ~Communicator();
  Communicator(const Communicator&) = delete;
  Communicator& operator=(const Communicator&) = delete;
  int world() const { return world_; }
  int rank() const { return rank_; }
  // NCCL all-gather of `bytes` from every rank into recv [world][bytes].
  void all_gather(const void* send_dev, void* recv_dev, std::size_t bytes, void* stream);
  void* raw() const { return comm_; }

 private:
  void* comm_ = nullptr;
  int world_ = 1, rank_ = 0;
};

// This rank's column shard of a [k][n] weight matrix (host inputs describe
// the FULL matrix; only the shard is uploaded).
class ShardedWeights {
 public:
  // max_m: largest row count the fused (peer-store) path will be called with
  // (sizes its double-buffered output arena; the NCCL path has no limit).
  ShardedWeights(Communicator& comm, const std::vector<std::uint8_t>& indices,
                 const std::vector<Half>& scales, const LookupTable& table, int k, int n,
                 const QuantConfig& cfg, int max_m = 32);
  ~ShardedWeights();
  ShardedWeights(const ShardedWeights&) = delete;
  ShardedWeights& operator=(const ShardedWeights&) = delete;

  int n0() const;
  int n1() const;
  DeviceWeights& local();

  // Y [m][n] on every rank: shard GEMM into a [m][n1-n0] slice, NCCL
  // all-gather, column re-layout (none for m = 1 with equal slices).
  void gemm(const Half* x_dev, int m, Half* y_dev, void* stream = nullptr);
  // Fused all-gather: the GEMM epilogue stores this rank's columns straight
  // into every rank's Y (CUDA IPC peer mappings over NVLink), then a device
  // flag barrier (release/acquire at system scope, no host round trip).  The
  // output arena is double-buffered, so no barrier precedes the GEMM.
  // Returns the device pointer of the full Y [m][n] on this rank; it stays
  // valid until the call after next.
  const Half* gemm_fused(const Half* x_dev, int m, void* stream = nullptr);

  struct Impl;

 private:
  std::unique_ptr<Impl> impl_;
};

}  // namespace flutesim
