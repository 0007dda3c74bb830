/* flute-b200 — C ABI of the B200 LUT-GEMM hot path.
 *
 * Plain C, plain pointers and sizes, no torch / CUDA types in the signatures
 * (streams are passed as void* = cudaStream_t).  Every entry point names the
 * reference interface it replaces (reference tree: /root/reference/proj).
 *
 * Status codes mirror the reference's exception taxonomy (errors.hpp:12-50):
 *   FLUTE_OK, FLUTE_ERR_CONFIG (ConfigError), FLUTE_ERR_INPUT (InputError),
 *   FLUTE_ERR_INTERNAL (InternalError), FLUTE_ERR_CUDA (CUDA runtime/driver),
 *   FLUTE_ERR_OPTIMIZATION (OptimizationError, refinement only).
 * flute_last_error() returns the message of the last failure on the calling
 * thread.  Nothing here falls back to the CPU: device entry points fail with
 * FLUTE_ERR_CUDA when no sm_100 device is usable.
 *
 * Index/scale/table conventions (quantize.hpp:17-39, vec_lut.hpp:18-30):
 *   indices  u8  [k][n] row-major, each < 2^bits
 *   scales   f16 [n][k/group] (column-major over groups), as raw u16 bits
 *   table    2^bits f32 values (narrowed to f16 exactly as the reference does)
 *   vLUT     2^(2*bits) u32 words: low half = T[i] (even k), high = T[j]
 *   x        f16 [m][k] row-major; y f16 [m][n] row-major
 */
#ifndef FLUTE_C_H
#define FLUTE_C_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FLUTE_OK 0
#define FLUTE_ERR_CONFIG 1
#define FLUTE_ERR_INPUT 2
#define FLUTE_ERR_INTERNAL 3
#define FLUTE_ERR_CUDA 4
#define FLUTE_ERR_OPTIMIZATION 5

const char* flute_last_error(void);
const char* flute_version(void);

/* ---- numerics (half.hpp:81-93) ------------------------------------------ */
uint16_t flute_f32_to_f16(float x);
float flute_f16_to_f32(uint16_t h);

/* ---- input producers (nf_table.hpp:48, quantize.hpp:45-52) --------------- */
int flute_nf_table(int bits, float* values_out /* 2^bits */);
/* nf_table.hpp:23-25: raw quantiles Phi^-1(p_i) (2^bits doubles) and sigma. */
int flute_nf_quantiles(int bits, double* values_out);
double flute_nf_sigma(void);
int flute_quantize(const float* w /* k x n */, int k, int n, int bits, int group,
                   uint8_t* indices_out, uint16_t* scales_out);

/* ---- canonical packer: reorder_and_split / unpack_matrix (pack.hpp:72-85) */
/* layout = {tile_m, tile_n, tile_k, frag_m, frag_n, frag_k} (pack.hpp:20-37).
 * slice_hi holds ceil(k*n*w/32) words (w = 2 for 3-bit, else bits); slice_lo
 * (3-bit only, may be NULL otherwise) holds ceil(k*n/32) words. */
size_t flute_canonical_words(int k, int n, int slice_bits);
int flute_pack_canonical(const uint8_t* indices, int k, int n, int bits, const int* layout,
                         uint32_t* slice_hi, uint32_t* slice_lo);
int flute_unpack_canonical(const uint32_t* slice_hi, const uint32_t* slice_lo, int k, int n,
                           int bits, const int* layout, uint8_t* indices_out);

/* ---- sm_100a device layout (new) --------------------------- */
int flute_device_sizes(int k, int n, int bits, int group, size_t* weight_bytes,
                       size_t* scale_bytes);
int flute_pack_device(const uint8_t* indices, int k, int n, int bits, int group,
                      uint8_t* out /* weight_bytes */);
int flute_repack_canonical(const uint32_t* slice_hi, const uint32_t* slice_lo, int k, int n,
                           int bits, const int* layout, int group, uint8_t* out);
int flute_unpack_device(const uint8_t* packed, int k, int n, int bits, int group,
                        uint8_t* indices_out);
int flute_scales_device(const uint16_t* scales, int k, int n, int group,
                        uint16_t* out /* scale_bytes/2 */);

/* ---- vectorized LUT: make_vectorized_lut / vec_dequantize (vec_lut.hpp:34-43) */
/* out: 2^(2b)*dup words, copy c of entry e at e*dup + c. */
int flute_vlut_build(const float* table_values, int bits, int dup, uint32_t* out);
/* dup-1 vLUT -> the 2^(2b) words in device-index order (identity for 2/4-bit). */
int flute_vlut_device_words(const uint32_t* vlut_words, int bits, uint32_t* out);
int flute_vec_dequantize(uint32_t pair, uint16_t scale, const uint32_t* vlut_words, int bits,
                         uint32_t* out /* first | second << 16 */);

/* ---- Stream-K plan (streamk.hpp:58) + traffic model (engine.hpp:74-96) --- */
/* ranges: 2*workers; fixups (nullable): 4 per split tile {tile, finisher,
 * slot_base, n_contributors}. */
int flute_plan_stream_k(int tiles_m, int tiles_n, int tiles_k, int workers, int64_t* ranges,
                        int64_t* fixups, int max_fixups, int* n_fixups, int64_t* total_slots);
/* stats: {weights, scales, table, activations, partials_rw, output, flops}. */
int flute_plan_traffic(int m, int k, int n, int bits, int group, const int* layout, int workers,
                       int stages, int tile_m, uint64_t* stats);
double flute_bits_per_param(int bits, int group);

/* ---- device: the qgemm (engine.hpp:72 execute, "qgemm" of the paper) ----- */
int flute_device_count(void);
int flute_sm_count(int device);
/* Largest Stream-K CTA count that is guaranteed co-resident for an m-row call
 * at any bit width (W2/W3 with 17..32 rows allow twice this); larger counts
 * are legal (ticketed worker ids keep the handshake deadlock-free). */
int flute_max_workers(int m);
/* Default worker count (CTAs) for a shape. */
int flute_default_workers(int m, int k, int n, int bits);

/* Raw device-pointer GEMM.  w / scales in device layout, vlut = the 2^(2b)
 * device-order words, all in device memory.  workspace: >=
 * flute_workspace_bytes(m, workers) bytes of device memory, zero-filled
 * before first use (the kernel leaves it zeroed).  One workspace must not be
 * used by two launches that may run concurrently.  workers <= 0 picks the
 * default.  Async on `stream` (cudaStream_t; NULL = legacy default). */
size_t flute_workspace_bytes(int m, int workers);
int flute_qgemm(const void* x, int m, int k, int n, const void* w, const void* scales,
                const void* vlut, int bits, int group, void* y, void* workspace,
                size_t workspace_bytes, int workers, void* stream);

/* Device-resident weight handle: uploads device-layout weights, scales and the
 * vLUT once (flute_weights_create*), owns a workspace. */
typedef struct flute_weights flute_weights;
int flute_weights_create(const uint8_t* packed_host, const uint16_t* scales_dev_layout_host,
                         const uint32_t* vlut_words /* dup 1, reference order */, int k, int n,
                         int bits, int group, flute_weights** out);
/* Convenience: from indices [k][n] + scales [n][k/g] + table values. */
int flute_weights_from_indices(const uint8_t* indices, const uint16_t* scales,
                               const float* table_values, int k, int n, int bits, int group,
                               flute_weights** out);
int flute_weights_destroy(flute_weights* w);
/* Pre-size the handle's device workspace for calls with m <= max_m so that no
 * later flute_gemm allocates (required before CUDA-graph capture of m > 32). */
int flute_weights_reserve(flute_weights* w, int max_m);
/* Time the candidate work decompositions (cluster split-K sizes, Stream-K CTA
 * counts) for m-row calls (1 <= m <= 32) on this handle's shape, L2 flushed
 * between runs, and keep the fastest for later workers <= 0 calls of the same
 * row class; `report` (nullable) receives the timings. */
int flute_weights_autotune(flute_weights* w, int m, void* stream, char* report, size_t cap);
int flute_weights_info(const flute_weights* w, int* k, int* n, int* bits, int* group);
int flute_gemm(flute_weights* w, const void* x_dev, int m, void* y_dev, int workers,
               void* stream);
/* End-to-end: x and y are HOST pointers; copies in, GEMM, copies out, syncs. */
int flute_gemm_host(flute_weights* w, const uint16_t* x_host, int m, uint16_t* y_host,
                    int workers, void* stream);
/* A batch of `count` end-to-end GEMMs (handle ws[i], host x_host[i] [m[i]][k_i]
 * -> host y_host[i] [m[i]][n_i]; a handle may repeat).  Input copies, GEMMs (on
 * `stream`) and output copies are pipelined over three streams; returns when
 * every output is in host memory.  Pinned host buffers make the copies DMA. */
int flute_gemm_host_batch(flute_weights* const* ws, const uint16_t* const* x_host, const int* m,
                          uint16_t* const* y_host, int count, int workers, void* stream);
/* The same batch prepared once and captured as a CUDA graph (copies in, GEMMs,
 * copies out, with their cross-stream dependencies; own staging buffers).
 * flute_host_batch_run replays it on `stream` and returns when every output
 * is in host memory.  The handles and host buffers must outlive the batch;
 * refill the inputs in place between runs. */
typedef struct flute_host_batch flute_host_batch;
int flute_host_batch_create(flute_weights* const* ws, const uint16_t* const* x_host, const int* m,
                            uint16_t* const* y_host, int count, int workers,
                            flute_host_batch** out);
int flute_host_batch_run(flute_host_batch* b, void* stream);
void flute_host_batch_destroy(flute_host_batch* b);

/* ---- weight preparation on the device / FLTE ----------
 * flute_quantize_device: quantize_matrix (quantize.cpp:81-128) on the GPU for
 * a device f32 [k][n] matrix -> device indices [k][n] u8 + binary16 scales
 * [n][k/g]; bit-exact with the host quantizer; synchronises `stream`.
 * flute_weights_from_device: a weight handle from device-resident indices +
 * scales (packed into the device layout on the GPU); table16 = 2^bits binary16.
 * flute_flte_info / flute_weights_from_flte: parse an FLTE container
 * (flte.hpp:4-9, strict, FLUTE_ERR_INPUT with section + byte offset on a bad
 * file) and upload it, canonical slices re-permuted on the GPU.
 * flute_flte_write: indices + scales + table -> FLTE bytes (reorder_and_split
 * at `layout`); out may be NULL to query *len. */
int flute_quantize_device(const float* w_dev, int k, int n, int bits, int group, uint8_t* idx_dev,
                          uint16_t* scales_dev, void* stream);
int flute_weights_from_device(const uint8_t* idx_dev, const uint16_t* scales_dev,
                              const uint16_t* table16, int k, int n, int bits, int group,
                              void* stream, flute_weights** out);
int flute_flte_info(const uint8_t* bytes, size_t len, int* bits, int* group, int* k, int* n);
int flute_weights_from_flte(const uint8_t* bytes, size_t len, void* stream, flute_weights** out);
int flute_flte_write(const uint8_t* indices, const uint16_t* scales, const float* table_values,
                     int k, int n, int bits, int group, const int* layout, uint8_t* out, size_t cap,
                     size_t* len);

/* ---- learned-sigma refinement --------------------
 * flute_ste_evaluate: ste_evaluate (quantize.cpp:141-229) on the GPU.  HOST
 * buffers: w f32 [k][n], x f32 [m][k] (calibration rows), sigma f64 [n*k/g]
 * ([n][k/g] group order); out: *loss, grad f64 [n*k/g], idx u8 [k][n] (grad /
 * idx may be NULL).  Indices and gradients are bit-identical to the
 * reference; the loss equals it up to summation order.
 * flute_refine_scales: refine_scales (quantize.cpp:231-282): `steps` descent
 * steps at rate `lr` on the GPU; out: idx u8 [k][n], scales f16 [n][k/g]
 * (learned factor folded in), sigma f64 [n*k/g] (may be NULL), losses[2] =
 * {initial, final} (may be NULL).  FLUTE_ERR_OPTIMIZATION when the loss or a
 * folded scale goes non-finite; *failed_step (may be NULL) = its step. */
int flute_ste_evaluate(const float* w, const float* x, int m, int k, int n, int bits, int group,
                       const double* sigma, double* loss, double* grad, uint8_t* idx);
int flute_refine_scales(const float* w, const float* x, int m, int k, int n, int bits, int group,
                        int steps, double lr, uint8_t* idx, uint16_t* scales, double* sigma,
                        double* losses, int* failed_step);

/* ---- N-column sharding ---------------------------------
 * Rank `rank` of `world` owns the 64-column tiles [rank*T/world,
 * (rank+1)*T/world) of T = ceil(n/64): columns [n0, n1).  Its device-layout
 * weights / scales are the contiguous byte ranges [w_off, w_off+w_bytes) /
 * [s_off, s_off+s_bytes) of the full buffers (any output may be NULL). */
int flute_shard_range(int k, int n, int bits, int group, int world, int rank, int* n0, int* n1,
                      size_t* w_off, size_t* w_bytes, size_t* s_off, size_t* s_bytes);
/* The all-gather fused into the epilogue: like flute_qgemm, but every output
 * value is stored to each of y_peers[0..n_peers) (device pointers reachable
 * from this GPU: NVLink peer or multicast mappings; n_peers <= 8) at
 * [row * ldy + ycol0 + col].  A rank passes its column offset n0 as ycol0 and
 * the full N as ldy; after a cross-rank barrier every rank holds the full Y. */
int flute_qgemm_peers(const void* x, int m, int k, int n, const void* w, const void* scales,
                      const void* vlut, int bits, int group, void* const* y_peers, int n_peers,
                      int ldy, int ycol0, void* workspace, size_t workspace_bytes, int workers,
                      void* stream);
int flute_gemm_peers(flute_weights* w, const void* x_dev, int m, void* const* y_peers, int n_peers,
                     int ldy, int ycol0, int workers, void* stream);

/* The N-sharded layer over the GPUs of one node, C++ host side
 * (include/flutesim/sharded.hpp; no reference counterpart — the reference is
 * one CPU process; each shard is its engine.cpp:345 GEMM on a column slice).
 * NCCL is loaded at run time (libnccl.so.2 already in the process, else the
 * system one).  Rank 0 calls flute_comm_unique_id and distributes the 128
 * bytes out of band; every rank then calls flute_comm_create on its GPU. */
#define FLUTE_COMM_ID_BYTES 128
typedef struct flute_comm flute_comm;
int flute_comm_unique_id(uint8_t* id_out /* FLUTE_COMM_ID_BYTES */);
int flute_comm_create(const uint8_t* id, int world, int rank, flute_comm** out);
int flute_comm_destroy(flute_comm* c);
typedef struct flute_sharded flute_sharded;
/* This rank's column shard of the FULL [k][n] matrix (host indices [k][n],
 * scales [n][k/g], table values); max_m bounds flute_sharded_gemm_fused. */
int flute_sharded_create(flute_comm* c, const uint8_t* indices, const uint16_t* scales,
                         const float* table_values, int k, int n, int bits, int group, int max_m,
                         flute_sharded** out);
int flute_sharded_destroy(flute_sharded* s);
int flute_sharded_info(const flute_sharded* s, int* n0, int* n1);
/* y_dev [m][n] (full Y on every rank): shard GEMM + ncclAllGather + re-layout. */
int flute_sharded_gemm(flute_sharded* s, const void* x_dev, int m, void* y_dev, void* stream);
/* Fused: the GEMM epilogue stores this rank's columns into every rank's
 * double-buffered output arena (CUDA IPC peer mappings), then a device
 * release/acquire flag barrier; *y_out = this rank's full Y [m][n], valid
 * until the call after next. */
int flute_sharded_gemm_fused(flute_sharded* s, const void* x_dev, int m, const void** y_out,
                             void* stream);

/* The reference call itself: flutesim::execute (engine.hpp:72, engine.cpp:345)
 * on HOST buffers in the reference's canonical formats — x f16 [m][k],
 * canonical slices from reorder_and_split at `layout`, scales f16 [n][k/g],
 * the make_vectorized_lut table (2^(2b)*dup words) — run on the GPU.  y:
 * f16 [m][n]; stats (nullable): the 7 TrafficStats fields of the reference
 * accounting model (== flute_plan_traffic for the same shape).  workers = the
 * Stream-K CTA count (the reference's simulated SMs); stages / tile_m are
 * validated as the reference does and never change results. */
int flute_execute(const uint16_t* x, int m, const uint32_t* slice_hi, const uint32_t* slice_lo,
                  int k, int n, int bits, int group, const int* layout, const uint16_t* scales,
                  const uint32_t* vlut_words, int dup, int workers, int stages, int tile_m,
                  uint16_t* y, uint64_t* stats);

/* ---- device self-checks (used by the parity tests) ----------------------- */
/* Run the kernel's own dequant routine over every pair x every scale:
 * out[s * 2^(2b) + p] = device half2 for (pair p, scales[s]); pair p in
 * reference order (the routine applies the device index permutation). */
int flute_dequant_all_device(const uint32_t* vlut_words, int bits, const uint16_t* scales,
                             int n_scales, uint32_t* out_host);
/* Diagnostics (libflute_b200_diag.so only; `make diag`): with
 * FLUTE_DEBUG_TIMES=1, each qgemm launch records per-CTA %globaltimer stamps
 * (ns) {start, producer issued, LUT ready, first stage landed, segment end,
 * last segment end, exit, finisher acquired} plus {after the CTA barrier,
 * producer policy set, producer PDL wait done, vLUT filled, epilogue PDL wait
 * done} (16*workers values) followed by a per-stage trace of consumer warp 0
 * (workers*64*3 values: wait begin, data ready, compute done); copies all
 * 208*workers values of the last launch. */
int flute_debug_times(uint64_t* out, int workers);
/* mma_fragment on the tensor cores (mma.hpp:23); host buffers. */
int flute_mma_fragment(const uint16_t* a, const uint16_t* b, float* c, int m, int n, int k);

#ifdef __cplusplus
}
#endif
#endif /* FLUTE_C_H */
