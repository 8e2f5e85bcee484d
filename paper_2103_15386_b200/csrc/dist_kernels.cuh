// dist_kernels.cuh -- kernels of the distributed GGM refine (SURVEY.md
// section 8(e) stage B).
//
// A tree level merges a group of G ranks; rank j of the group owns the lists
// of the group-local ids [j n_l, (j+1) n_l) (its own shard), the group's
// vectors are replicated, and one restricted iteration
// becomes, on every rank, over its own nodes only:
//   k_merge_sample (unchanged; S.fpos == nullptr: no local reverse counts)
//   -> k_fwd_count / k_fwd_scatter: forward samples as reverse records
//      (target, source) grouped by the target's owner  -> exchange
//   -> k_rec_count / k_rec_scatter: the owner's reverse CSR
//   -> k_scan_*, k_rev_select (unchanged, node ids D.base + v)
//   -> join in record mode: (target, key) records, thresholds from the
//      gathered k-th keys (D17)
//   -> k_cand_count / k_cand_scatter: records grouped by owner -> exchange
//   -> k_cand_apply: the owner files them into its buckets (D34 capacity).
// Every step is bulk-synchronous and order-independent (D10, D17), so the
// result equals the one-GPU merge bit for bit.
#pragma once
#include "graph_kernels.cuh"

namespace knng {

__global__ void k_flag_shift(int* f) { *f = *f ? 2 : 0; }

// key ids shifted by delta (the group's first global id: global <-> local)
__global__ void k_keys_shift(uint64_t* __restrict__ keys, int64_t total, int64_t delta) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= total) return;
    const uint64_t kk = keys[i];
    if (kk == kSentinel) return;
    keys[i] = (kk & 0xFFFFFFFF00000000ull) | static_cast<uint32_t>(static_cast<int64_t>(key_id(kk)) + delta);
}

// (ids, dists) of a built shard -> keys with ids + delta
__global__ void k_to_keys(const uint32_t* __restrict__ ids, const float* __restrict__ dists, int64_t total,
                          int64_t delta, uint64_t* __restrict__ keys) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= total) return;
    keys[i] = make_key(dists[i], static_cast<uint32_t>(static_cast<int64_t>(ids[i]) + delta));
}

// Reverse records: forward sample (s, j) of flag f whose target v (a group id)
// is owned by group rank v / n_l.  Record = (v - owner n_l) | f << 31, then
// the source's group id D.base + s.  Pass 1 counts per (owner, flag) and keeps
// each record's position inside its bin (S.fpos, free in this mode).
__global__ void k_fwd_count(Dims D, Samples S, uint32_t* __restrict__ pos, int64_t n_l,
                            unsigned int* __restrict__ cnt) {
    const int f = blockIdx.y;
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= D.n * D.p) return;
    const int64_t s = i / D.p;
    const int j = static_cast<int>(i - s * D.p);
    if (j >= S.fcnt[2 * s + f]) return;
    const uint32_t v = S.fwd[static_cast<size_t>(f) * D.n * D.p + i];
    const int owner = static_cast<int>(v / n_l);
    pos[static_cast<size_t>(f) * D.n * D.p + i] = atomicAdd(cnt + 2 * owner + f, 1u);
}
// Pass 2: record of bin (owner, f) goes to binoff[2 owner + f] + its position
// (records of one owner: flag 0 then flag 1, contiguous).
__global__ void k_fwd_scatter(Dims D, Samples S, const uint32_t* __restrict__ pos, int64_t n_l,
                              const unsigned long long* __restrict__ binoff, uint2* __restrict__ out) {
    const int f = blockIdx.y;
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= D.n * D.p) return;
    const int64_t s = i / D.p;
    const int j = static_cast<int>(i - s * D.p);
    if (j >= S.fcnt[2 * s + f]) return;
    const uint32_t v = S.fwd[static_cast<size_t>(f) * D.n * D.p + i];
    const int owner = static_cast<int>(v / n_l);
    const uint32_t vl = static_cast<uint32_t>(v - static_cast<int64_t>(owner) * n_l);
    out[binoff[2 * owner + f] + pos[static_cast<size_t>(f) * D.n * D.p + i]] =
        make_uint2(vl | (static_cast<uint32_t>(f) << 31), static_cast<uint32_t>(D.base + s));
}

// Owner side: reverse counts (the slot is the count's old value), then the
// CSR scatter once k_scan_* has turned the counts into offsets.
__global__ void k_rec_count(const uint2* __restrict__ rec, int64_t nrec, Samples S, int64_t n,
                            uint32_t* __restrict__ rpos) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= nrec) return;
    const uint32_t w = rec[i].x;
    const int f = static_cast<int>(w >> 31);
    rpos[i] = atomicAdd(S.rcnt + f * n + (w & 0x7FFFFFFFu), 1u);
}
__global__ void k_rec_scatter(const uint2* __restrict__ rec, int64_t nrec, Samples S, int64_t n,
                              int64_t rstride, const uint32_t* __restrict__ rpos) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= nrec) return;
    const uint2 r = rec[i];
    const int f = static_cast<int>(r.x >> 31);
    const uint32_t v = r.x & 0x7FFFFFFFu;
    S.rsrc[static_cast<size_t>(f) * rstride + S.off[f * (n + 1) + v] + rpos[i]] = r.y;
}

// Candidate records of the joins (record mode) grouped by the target's owner.
struct CandRec {
    uint64_t key;
    uint32_t tgt;  // owner-local node index
    uint32_t pad;
};
__global__ void k_cand_count(const uint32_t* __restrict__ tgt, const unsigned long long* __restrict__ nrec,
                             int64_t n_l, uint32_t* __restrict__ pos, unsigned int* __restrict__ cnt) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= static_cast<int64_t>(*nrec)) return;
    pos[i] = atomicAdd(cnt + tgt[i] / n_l, 1u);
}
__global__ void k_cand_scatter_owner(const uint32_t* __restrict__ tgt, const uint64_t* __restrict__ key,
                                     const unsigned long long* __restrict__ nrec, int64_t n_l,
                                     const uint32_t* __restrict__ pos, const unsigned long long* __restrict__ binoff,
                                     CandRec* __restrict__ out) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= static_cast<int64_t>(*nrec)) return;
    const uint32_t t = tgt[i];
    const int owner = static_cast<int>(t / n_l);
    out[binoff[owner] + pos[i]] = CandRec{key[i], static_cast<uint32_t>(t - static_cast<int64_t>(owner) * n_l), 0u};
}
// owner: file the received records into its buckets (already below the
// target's k-th key: the senders filtered with the gathered thresholds)
__global__ void k_cand_apply(const CandRec* __restrict__ rec, int64_t nrec, Graph G) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= nrec) return;
    const CandRec r = rec[i];
    const uint32_t slot = atomicAdd(G.bcnt + r.tgt, 1u);
    G.bucket[G.boff[r.tgt] + slot] = r.key;
}

}  // namespace knng
