/*
 * knng_oracle.h -- TEST INFRASTRUCTURE ONLY (parity oracle), not product code.
 *
 * A plain, slow, single-threaded C99 reference of GNND, the GPU redesign of
 * NN-Descent in Wang, Zhao, Zeng, "Large-Scale Approximate k-NN Graph
 * Construction on GPU" (arXiv 2103.15386).  Citation key: "P:n" is line n of
 * the paper text (/root/reference/PAPER.md at survey time); "Dn" is reading n
 * of the ambiguity ledger in DESIGN.md section 3.
 *
 * Who may use it: only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs.  The CUDA product path never links,
 * loads or calls anything here, and this file shares no code with it (its
 * Philox, metrics, sampling, join and update are written independently).
 *
 * Data conventions (identical by DEFINITION to the product ABI, not by code):
 *   key(d, id) = (float_bits(d) << 32) | id   (u64; d >= +0 so the bit order
 *                is the order of (d, id) lexicographically -- D3)
 *   keys  : u64 [n][k]  each list ascending
 *   flags : u8  [n][k]  1 = NEW, 0 = OLD
 *   SENTINEL = 0xFFFFFFFFFFFFFFFF  -- the (inf, inf) tuple of Alg. 2
 *
 * Parity pins: see tests/test_oracle_*.py (Philox known answers, SPEC worked
 * examples, brute force on tiny inputs, invariants, closed forms).
 */
#ifndef KNNG_ORACLE_H
#define KNNG_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_OK = 0, ORC_E_USAGE = 1, ORC_E_DOMAIN = 2, ORC_E_NOMEM = 3 };
enum { ORC_L2SQ = 0, ORC_COSINE = 1, ORC_CHI2 = 2 };
enum { ORC_UPDATE_SELECTIVE = 0, ORC_UPDATE_FULL = 1 };
enum { ORC_F32 = 0, ORC_U8 = 1 };

/* Philox counter tags (D31) */
enum { ORC_TAG_INIT = 1, ORC_TAG_REV_NEW = 2, ORC_TAG_REV_OLD = 3,
       ORC_TAG_MERGE_SEED = 4 };

#define ORC_SENTINEL 0xFFFFFFFFFFFFFFFFull

typedef struct {
    int64_t dist_evals;  /* pairs whose distance was computed            */
    int64_t candidates;  /* non-sentinel GetNearestObject results offered */
    int64_t accepted;    /* list entries that are new after the update    */
    int64_t joins;       /* local joins run (nodes with m > 0)            */
    int64_t sum_m;       /* sum over joins of |G_new(x)|                   */
    int64_t sum_q;       /* sum over joins of |G_old(x)|                   */
} orc_stats;

/* Philox4x32-10 (Salmon et al., SC'11; the generator cuRAND calls
 * Philox4_32_10).  ctr = 4 words, key = 2 words. */
void orc_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2],
                       uint32_t out[4]);
/* uniform integer in [0, N): (u64(out1:out0) * N) >> 64  (D31) */
uint64_t orc_uniform(const uint32_t out[4], uint64_t N);

/* Options (process-wide, test infrastructure):
 *   "update"        ORC_UPDATE_SELECTIVE (GNND, Alg. 2: the nearest object
 *                   of each sample) or ORC_UPDATE_FULL (GNND-r1,
 *                   every produced pair offered to its lists)
 *   "segment_size"  entries per list segment (32); lists with k >=
 *                   2 * segment_size are split into k / segment_size
 *                   segments (D40); smaller k: one segment (D18). */
int orc_set_option(const char* name, int value);
int orc_segments(int k);  /* segment count of a k-list; -1 if k is not a multiple */
/* Segmented InsertIntoNNList: list = sorted union of s
 * segments, id v in segment v % s.  Returns 1 if inserted, -1 usage. */
int orc_list_insert_seg(uint64_t* list, uint8_t* flags, int k, int s, uint64_t key);

/* Canonical distance between rows a and b (D4, D5, D6, D39 chi-square). */
float orc_distance(const void* X, int dtype, int64_t n, int d, int metric,
                   int64_t a, int64_t b);

/* Eq. 1-2: thread t of the NEW-NEW block computes the pair
 * (u, v), u = ceil(sqrt(2t + 2.25) - 0.5), v = t - u(u-1)/2, stored at
 * D_new[u(u-1)/2 + v].  fp64 evaluation. */
void orc_pair_index(int64_t t, int64_t* u, int64_t* v);

/* InsertIntoNNList on one bounded sorted list (D16); returns 1 if
 * inserted.  Exposed for the SPEC S:86-88 worked examples. */
int orc_list_insert(uint64_t* list, uint8_t* flags, int k, uint64_t key);

/* Alg. 1 lines 1-4: k distinct random neighbours != s, sorted,
 * all NEW. */
int orc_init(const void* X, int dtype, int64_t n, int d, int metric, int k,
             uint64_t seed, uint64_t* keys, uint8_t* flags);

/* ParallelSample with the readings D7-D11.  Pure: does
 * not modify keys/flags.  Outputs (any may be NULL):
 *   FN/FO  [n][p]  forward NEW / OLD samples, counts fnc/foc
 *   Gn/Go  [n][2p] sorted unique sample lists, counts cn/co (Go excludes Gn)
 * tword: the iteration word of the reverse-priority counter. */
int orc_sample(int64_t n, int k, int p, uint32_t tword, uint64_t seed,
               const uint64_t* keys, const uint8_t* flags,
               uint32_t* FN, int32_t* fnc, uint32_t* FO, int32_t* foc,
               uint32_t* Gn, int32_t* cn, uint32_t* Go, int32_t* co);

/* One GNND iteration (Alg. 1 lines 8-31): sample, local join
 * with selective update (Alg. 2), immediate InsertIntoNNList in join
 * order, then "mark all sampled neighbours OLD".
 * boundary < 0: plain build; boundary >= 0: GGM refine, pairs (a, b) with
 *   (a >= boundary) == (b >= boundary) are skipped (D22).
 * target_mask: NULL = update every list; else only lists t with mask[t] != 0
 *   are updated (and only joins touching a target are run) -- the same
 *   definition evaluated on a subset of outputs, for full-size parity. */
int orc_iterate(const void* X, int dtype, int64_t n, int d, int metric, int k,
                int p, uint32_t tword, uint64_t seed, int64_t boundary,
                uint64_t* keys, uint8_t* flags, const uint8_t* target_mask,
                orc_stats* st);

/* ConstructKNNGraph (Alg. 1): init + exactly iters iterations (D20).
 * out_ids/out_dists [n][k]; per_iter: iters entries or NULL. */
int orc_build(const void* X, int dtype, int64_t n, int d, int metric, int k,
              int p, int iters, uint64_t seed, uint32_t* out_ids,
              float* out_dists, orc_stats* per_iter);

/* GGM (Alg. 3) on the combined set: rows [0, nA) are S1, rows
 * [nA, n) are S2; keys_in holds both graphs with S2 ids already re-based.
 *   seed step  : keep first ceil(k/2) (OLD), reserve last floor(k/2),
 *                draw floor(k/2) distinct ids of the other subset (NEW).
 *   refine     : merge_iters restricted iterations (boundary = nA).
 *   finalize   : k smallest unique of refined list U reserved.
 * level: tree level, part of the seed-draw counter (D26). */
int orc_ggm_seed(const void* X, int dtype, int64_t n, int d, int metric,
                 int k, int64_t nA, int level, uint64_t seed,
                 const uint64_t* keys_in, uint64_t* keys, uint8_t* flags,
                 uint64_t* reserved);
int orc_ggm_finalize(int64_t n, int k, const uint64_t* reserved,
                     uint64_t* keys);
int orc_merge(const void* X, int dtype, int64_t n, int d, int metric, int k,
              int p, int64_t nA, int merge_iters, int level, uint64_t seed,
              const uint64_t* keys_in, uint64_t* keys_out,
              orc_stats* per_iter);

/* Exact top-kq by key over j != q ("exhaustive"), for queries[nq]. */
int orc_bruteforce(const void* X, int dtype, int64_t n, int d, int metric,
                   const int64_t* queries, int64_t nq, int kq,
                   uint64_t* out_keys);

/* Recall@k, Eq. 4 over the nq queries with the tie rule D27:
 * entry j of the graph's first at_k counts iff d(i, j) <= d_true_at_k(i).
 * graph_keys: [nq][kg] rows of the queried nodes; truth_keys: [nq][kt]. */
double orc_recall(int64_t nq, int kg, const uint64_t* graph_keys, int kt,
                  const uint64_t* truth_keys, int at_k);

/* phi(G), Eq. 3: fp64 sum of the stored distances. */
double orc_phi(int64_t n, int k, const uint64_t* keys);

#ifdef __cplusplus
}
#endif
#endif
