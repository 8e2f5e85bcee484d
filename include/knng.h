/*
 * knng.h -- C ABI of the B200-native GNND library (libknng.so).
 *
 * GNND is the GPU redesign of NN-Descent in Wang, Zhao, Zeng, "Large-Scale
 * Approximate k-NN Graph Construction on GPU" (arXiv 2103.15386).  "P:n"
 * cites line n of the paper text; "Dn" cites reading n of DESIGN.md section 3
 * (where the paper is silent or ambiguous).  The product is this library;
 * the Python module paper_2103_15386_b200.knng only marshals arguments.
 *
 * Conventions shared by every entry point
 * ---------------------------------------
 *  - Pointers are DEVICE pointers (cudaMalloc / torch CUDA tensors) unless
 *    the parameter name says host_.  The caller owns every buffer.
 *  - stream is a cudaStream_t passed as void* (NULL = legacy default stream).
 *    Every call enqueues on it and then BLOCKS until the stream work is done,
 *    so asynchronous CUDA faults are reported by the call that caused them.
 *  - Validation happens on the host before anything is enqueued: on a usage
 *    error nothing is written and KNNG_E_USAGE / KNNG_E_DOMAIN is returned.
 *    Parameter checks run before any CUDA API call, so they also work on a
 *    machine without a GPU.
 *  - No C++ exception crosses the ABI.  knng_last_error() returns a
 *    thread-local message for the last non-OK status.
 *  - Vectors are row-major [n][d]: float32 (KNNG_F32) or uint8 (KNNG_U8).
 *  - Graph output: out_ids u32 [n][k], out_dists f32 [n][k]; each list is
 *    sorted ascending by (dist, id) (D3).  Distances are squared L2 (D4) or
 *    1 - cos (D6), evaluated in the canonical order of D5/D6, so every stored
 *    distance equals a recomputed one bit for bit; u8 distances are exact
 *    integers stored as float.
 *  - Determinism: outputs are a pure function of (inputs, parameters, seed).
 *  - Limits of this version: 2 <= k <= 32, 1 <= sample_size(p) < k,
 *    2p <= 32 (p <= 16), n < 2^32 - 1, n > k, n * p < 2^32.
 */
#ifndef KNNG_H
#define KNNG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    KNNG_OK = 0,
    KNNG_E_USAGE = 1,    /* invalid argument; nothing was written            */
    KNNG_E_DOMAIN = 2,   /* input outside the metric's domain (zero vector
                            under cosine)                                    */
    KNNG_E_NOMEM = 3,    /* workspace too small / device allocation failed  */
    KNNG_E_CUDA = 4,     /* CUDA runtime error (message in knng_last_error) */
    KNNG_E_NCCL = 5,     /* reserved for the sharded build                  */
    KNNG_E_INTERNAL = 6
} knng_status;

typedef enum { KNNG_L2SQ = 0, KNNG_COSINE = 1 } knng_metric;
typedef enum { KNNG_F32 = 0, KNNG_U8 = 1 } knng_dtype;

/* Per-iteration counters of the device path (host struct). */
typedef struct {
    int64_t joins;        /* local joins run: nodes with |G_new| > 0          */
    int64_t sum_m;        /* sum of |G_new(x)| over joins                      */
    int64_t sum_q;        /* sum of |G_old(x)| over joins                      */
    int64_t dist_evals;   /* distances the method needs: m(m-1)/2 + m q per
                             join (only cross pairs in a GGM refine)           */
    int64_t candidates;   /* non-sentinel GetNearestObject results (Alg. 2)    */
    int64_t appended;     /* candidates below the target's k-th key (filed
                             into its bucket)                                */
    int64_t accepted;     /* list entries that are new after the update      */
    int64_t rows;         /* vector rows gathered by the join kernel          */
    int64_t recomputed;   /* canonical distance recomputations of the float
                             tensor-core join (its exact-selection window);
                             0 for the other join kernels                    */
} knng_iter_stats;

/* ------------------------------------------------------------------------
 * knng_build -- ConstructKNNGraph, Alg. 1: random init (P:98-103,
 * D1-D3), then exactly `iters` iterations (D20) of ParallelSample (P:145-151,
 * D7-D11), local join with selective update (Alg. 2) and the
 * bounded k-NN list update (D16-D17).
 *   vectors    [n][d] device, dtype dt
 *   k          neighbours per node; sample_size = p ("p < k")
 *   seed       key of every Philox draw (D31)
 *   out_ids    [n][k] device u32;  out_dists [n][k] device f32
 *   workspace  device scratch of >= knng_build_workspace_bytes(...) bytes,
 *              256-byte aligned (else KNNG_E_USAGE), or NULL with
 *              workspace_bytes == 0 to let the library allocate
 *              (cudaMallocAsync on `stream`) and free it before returning.
 * ---------------------------------------------------------------------- */
size_t knng_build_workspace_bytes(knng_dtype dt, int64_t n, int32_t d,
                                  int32_t k, int32_t sample_size,
                                  knng_metric metric);
knng_status knng_build(const void* vectors, knng_dtype dt, int64_t n,
                       int32_t d, int32_t k, knng_metric metric,
                       int32_t iters, int32_t sample_size, uint64_t seed,
                       uint32_t* out_ids, float* out_dists, void* workspace,
                       size_t workspace_bytes, void* stream);

/* Same computation with HOST buffers (pageable or pinned): copies the
 * vectors in, builds, copies the graph out.  The end-to-end entry point. */
knng_status knng_build_host(const void* host_vectors, knng_dtype dt,
                            int64_t n, int32_t d, int32_t k,
                            knng_metric metric, int32_t iters,
                            int32_t sample_size, uint64_t seed,
                            uint32_t* host_out_ids, float* host_out_dists,
                            void* stream);

/* ------------------------------------------------------------------------
 * knng_merge -- GGM, Alg. 3.  Graph A over vecA [nA][d] with
 * local ids, graph B over vecB [nB][d] with local ids (B's own numbering).
 * Output: (nA + nB) lists; ids of B are re-based by +nA.  Seed step keeps
 * ceil(k/2) entries (OLD), reserves floor(k/2), draws floor(k/2) distinct
 * ids of the other subset (NEW) with Philox counter (4, i, j, level) (D21,
 * D25); `merge_iters` GNND iterations restricted to cross pairs (P:288,
 * D22); final k smallest unique of refined U reserved.
 *   Requires nA, nB >= floor(k/2).  level: tree level (0 for a plain merge).
 * ---------------------------------------------------------------------- */
size_t knng_merge_workspace_bytes(knng_dtype dt, int64_t nA, int64_t nB,
                                  int32_t d, int32_t k, int32_t sample_size,
                                  knng_metric metric);
knng_status knng_merge(const void* vecA, int64_t nA, const uint32_t* idsA,
                       const float* distsA, const void* vecB, int64_t nB,
                       const uint32_t* idsB, const float* distsB,
                       knng_dtype dt, int32_t d, int32_t k,
                       knng_metric metric, int32_t merge_iters,
                       int32_t sample_size, int32_t level, uint64_t seed,
                       uint32_t* out_ids, float* out_dists, void* workspace,
                       size_t workspace_bytes, void* stream);

/* ------------------------------------------------------------------------
 * Sharded build (D26, D36, section 11).  There is no
 * separate C entry point: the multi-GPU build is knng_build on every shard
 * (shard g of S built with seed + g, local ids) followed by knng_merge per
 * tree level (level l merges groups of 2^(l+1) shards, ids numbered from the
 * group's first row, Philox level l).  The exchange between GPUs is one
 * point-to-point block transfer (vectors, ids, dists) per level, done by
 * paper_2103_15386_b200/sharded.py over torch.distributed (NCCL on NVLink);
 * knng_merge uses the received rows in place when they follow the leader's
 * own (D37).  The result depends only on S, not on the number of GPUs.
 * ---------------------------------------------------------------------- */

/* ------------------------------------------------------------------------
 * knng_bruteforce -- exact top-kq neighbours (j != q) of nq query rows by
 * exhaustive scan, for recall@10 ground truth (Eq. 4).
 *   queries [nq] device int64 row ids; out_ids/out_dists [nq][kq] device.
 *   1 <= kq <= 32, kq < n.
 * ---------------------------------------------------------------------- */
knng_status knng_bruteforce(const void* vectors, knng_dtype dt, int64_t n,
                            int32_t d, knng_metric metric,
                            const int64_t* queries, int64_t nq, int32_t kq,
                            uint32_t* out_ids, float* out_dists,
                            void* stream);

/* ------------------------------------------------------------------------
 * Debug / parity ABI (teacher forcing).  State format, as the oracle's:
 *   keys  u64 [n][k]: key = float_bits(dist) << 32 | id, ascending
 *   flags u8  [n][k]: 1 = NEW, 0 = OLD
 * All buffers device.  workspace as for knng_build (NULL/0 = allocate).
 * ---------------------------------------------------------------------- */
/* Alg. 1 lines 1-4: random init. */
knng_status knng_debug_init(const void* vectors, knng_dtype dt, int64_t n,
                            int32_t d, int32_t k, knng_metric metric,
                            uint64_t seed, uint64_t* keys, uint8_t* flags,
                            void* stream);
/* One iteration from (keys, flags), in place.  tword: the iteration word of
 * the reverse-sample Philox counter (t for a build; 0x80000000 | level << 16
 * | t for a GGM refine).  boundary < 0: plain; else GGM restriction.
 * host_stats (nullable) receives the iteration's counters. */
knng_status knng_debug_iterate(const void* vectors, knng_dtype dt,
                               int64_t n, int32_t d, int32_t k,
                               knng_metric metric, int32_t sample_size,
                               uint32_t tword, uint64_t seed,
                               int64_t boundary, uint64_t* keys,
                               uint8_t* flags, knng_iter_stats* host_stats,
                               void* workspace, size_t workspace_bytes,
                               void* stream);
/* ParallelSample only: Gn/Go [n][2p] (sorted unique ids, first cn/co valid),
 * cn/co [n] int32.  keys/flags are not modified. */
knng_status knng_debug_sample(int64_t n, int32_t k, int32_t sample_size,
                              uint32_t tword, uint64_t seed,
                              const uint64_t* keys, const uint8_t* flags,
                              uint32_t* Gn, int32_t* cn, uint32_t* Go,
                              int32_t* co, void* workspace,
                              size_t workspace_bytes, void* stream);
/* The device Philox4x32-10: out[i] = philox(ctr[i], key = seed), m blocks
 * of 4 words each (known-answer check of the device generator). */
knng_status knng_debug_philox(const uint32_t* ctr, int64_t m, uint64_t seed,
                              uint32_t* out, void* stream);

/* ------------------------------------------------------------------------
 * Options (process-wide; names are case-sensitive; unknown name ->
 * KNNG_E_USAGE).
 *   "exact_u8"     1 (default): float32 input under KNNG_L2SQ whose values
 *                  are all integers in [0, 255] and d <= 258 (so every
 *                  distance is an exact integer < 2^24) is copied once to
 *                  uint8 and built on the integer path.  Every distance is
 *                  then the same exact integer the canonical fp32 evaluation
 *                  (D5) yields, so the graph is bit-identical; SIFT-like data
 *                  qualifies.  0: always use the float path.
 *   "join_kernel"  0 (default): automatic -- the tensor-core join
 *                  (join_tc.cuh, exact int8 Gram tiles; 8 epilogue warps, 3
 *                  CTAs per SM; rows gathered by TMA gather4) for uint8 L2
 *                  rows of d <= 128, d % 16 == 0, else the warp-specialised
 *                  CUDA-core join (join_ws.cuh);
 *                  1: the batched cp.async join (join_kernel.cuh; also the
 *                     automatic choice for rows that are not 16-B aligned);
 *                  2: always the warp-specialised join;
 *                  4: float rows (L2 / cosine, d % 4 == 0, d <= 128): the
 *                     TF32 tensor-core join (join_tcf.cuh) -- exact
 *                     selection by canonical recomputation inside an
 *                     a-priori error window.
 *                  All produce bit-identical graphs.
 *   "last_exact_u8" (read-only) 1 if the last build/merge on this thread ran
 *                  on the exact integer path.
 * ---------------------------------------------------------------------- */
knng_status knng_set_option(const char* name, int64_t value);
knng_status knng_get_option(const char* name, int64_t* host_value);

/* ------------------------------------------------------------------------
 * Introspection
 * ---------------------------------------------------------------------- */
/* Counters of the iterations of the last build/merge on this thread (host):
 * copies min(max_iters, available) entries; returns the number copied. */
int32_t knng_last_stats(knng_iter_stats* host_out, int32_t max_iters);
/* Kernel launches issued by this library since load (all threads). */
int64_t knng_launch_count(void);
/* Per-kernel device timing with CUDA events on the launch stream.  When
 * enabled, every launch of the named kernels is bracketed by events and the
 * elapsed time accumulated; knng_kernel_time reads (ms total, launches). */
void knng_set_timing(int32_t enable);
void knng_reset_timing(void);
int32_t knng_kernel_time(const char* name, double* total_ms,
                         int64_t* launches);
const char* knng_last_error(void);
const char* knng_status_string(knng_status s);
int32_t knng_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* KNNG_H */
