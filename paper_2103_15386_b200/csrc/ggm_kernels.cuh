// ggm_kernels.cuh -- GGM graph merge, Alg. 3.  Warp per node of
// the combined set S = S1 U S2 (rows [0, nA) are S1, [nA, n) are S2).
#pragma once
#include "graph_kernels.cuh"

namespace knng {

// Seed (Alg. 3 lines 1-7): keep the first ceil(k/2)
// entries of the node's input list (OLD), reserve the last floor(k/2)
// (G^v), append floor(k/2) distinct ids of the other subset drawn
// in counter order from Philox(MERGE_SEED, i, j, level) (D21), NEW,
// then sort (D25).  Input lists must be ascending (as knng_build emits).
// One node's seed: `in` = its input entry in lane < k (ascending list);
// node i (an id of the merge's numbering, local index li of the launch)
// draws from the other subset [obase, obase + osize).
template <typename T, int MET>
__device__ __forceinline__ void ggm_seed_node(const T* __restrict__ X, const float* __restrict__ Xn, const Dims& D,
                                              int64_t li, int64_t i, uint64_t in, int64_t obase, uint64_t osize,
                                              int level, uint64_t seed, Graph& G, uint64_t* __restrict__ reserved) {
    const uint32_t lane = lane_id();
    const int k = D.k, kh = (k + 1) / 2, kr = k - kh;
    if (static_cast<int>(lane) >= kh && static_cast<int>(lane) < k)
        reserved[static_cast<size_t>(li) * kr + (lane - kh)] = in;
    // chosen ids: lanes [0, kh) keep their input entry; draws fill [kh, k)
    uint32_t chosen = static_cast<int>(lane) < kh ? key_id(in) : 0xFFFFFFFFu;
    const uint2 key = seed_key(seed);
    extern __shared__ uint32_t seed_scratch[];  // 32 u32 per warp
    uint32_t* scr = seed_scratch + (threadIdx.x >> 5) * 32;
    int cnt = kh;
    for (uint32_t j0 = 0; cnt < k; j0 += 32) {
        const uint4 o = philox4x32_10(
            make_uint4(kTagMergeSeed, static_cast<uint32_t>(i), j0 + lane, static_cast<uint32_t>(level)), key);
        const uint32_t v = static_cast<uint32_t>(obase + static_cast<int64_t>(uniform_below(o, osize)));
        bool dup = false;
        for (int t = 0; t < cnt; ++t) dup |= (__shfl_sync(kFull, chosen, t) == v);
        dup |= (__match_any_sync(kFull, v) & lanemask_lt()) != 0u;  // an earlier lane drew it
        const uint32_t acc = __ballot_sync(kFull, !dup);
        // accepted draw of rank r fills lane cnt + r (compaction through shared memory)
        __syncwarp();
        if (!dup && cnt + __popc(acc & lanemask_lt()) < k) scr[cnt + __popc(acc & lanemask_lt())] = v;
        __syncwarp();
        const int nc = min(k, cnt + __popc(acc));
        if (static_cast<int>(lane) >= cnt && static_cast<int>(lane) < nc) chosen = scr[lane];
        cnt = nc;
    }
    // (key << 1) | NEW: all k keys are distinct (kept own-subset entries and
    // cross draws), so the flag rides in bit 0 through the sorting network
    uint64_t e = kSentinel;
    if (static_cast<int>(lane) < kh) {
        e = in << 1;  // kept half: OLD
    } else if (static_cast<int>(lane) < k) {
        float dist;
        if constexpr (MET == kMetCos) {
            dist = Canon<float>::cos(Xn + static_cast<size_t>(i) * D.d, Xn + static_cast<size_t>(chosen) * D.d, D.d);
        } else if constexpr (MET == kMetChi2) {
            dist = Canon<float>::chi2(X + static_cast<size_t>(i) * D.d, X + static_cast<size_t>(chosen) * D.d, D.d);
        } else {
            dist = Canon<T>::l2(X + static_cast<size_t>(i) * D.d, X + static_cast<size_t>(chosen) * D.d, D.d);
        }
        e = (make_key(dist, chosen) << 1) | 1ull;  // cross sample: NEW
    }
    e = warp_sort_u64(e);
    const bool in_list = static_cast<int>(lane) < k;
    const uint64_t ek = e == kSentinel ? kSentinel : (e >> 1);
    if (in_list) G.keys[static_cast<size_t>(li) * k + lane] = ek;
    const uint32_t nm = __ballot_sync(kFull, in_list && (e & 1ull));
    if (lane == 0) G.newmask[li] = nm;
    if (static_cast<int>(lane) == k - 1) G.kth[li] = ek;
}

template <typename T, int MET>
__global__ void k_ggm_seed(const T* __restrict__ X, const float* __restrict__ Xn, Dims D, int64_t nA, int level,
                           uint64_t seed, const uint32_t* __restrict__ idsA, const float* __restrict__ distsA,
                           const uint32_t* __restrict__ idsB, const float* __restrict__ distsB, Graph G,
                           uint64_t* __restrict__ reserved, int* __restrict__ bad) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (i >= D.n) return;
    const uint32_t lane = lane_id();
    const int k = D.k;
    const bool own_b = i >= nA;
    uint64_t in = kSentinel;
    if (static_cast<int>(lane) < k) {
        // input ids must lie in their own graph's range (else KNNG_E_USAGE)
        if (!own_b) {
            const uint32_t id = idsA[static_cast<size_t>(i) * k + lane];
            if (id >= static_cast<uint64_t>(nA)) atomicExch(bad, 1);
            in = make_key(distsA[static_cast<size_t>(i) * k + lane], id);
        } else {
            const size_t o = static_cast<size_t>(i - nA) * k + lane;
            const uint32_t id = idsB[o];
            if (id >= static_cast<uint64_t>(D.n - nA)) atomicExch(bad, 1);
            in = make_key(distsB[o], static_cast<uint32_t>(id + nA));
        }
    }
    ggm_seed_node<T, MET>(X, Xn, D, i, i, in, own_b ? 0 : nA, static_cast<uint64_t>(own_b ? nA : D.n - nA), level,
                          seed, G, reserved);
}

// Distributed refine: the launch owns nodes D.base + [0, D.n) of a merge over
// n_all ids; keys_in holds their lists (merge-numbered ids, ascending).
template <typename T, int MET>
__global__ void k_ggm_seed_keys(const T* __restrict__ X, const float* __restrict__ Xn, Dims D, int64_t nA,
                                int64_t n_all, int level, uint64_t seed, const uint64_t* __restrict__ keys_in,
                                Graph G, uint64_t* __restrict__ reserved) {
    const int64_t li = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (li >= D.n) return;
    const int64_t i = D.base + li;
    const bool own_b = i >= nA;
    const uint64_t in = static_cast<int>(lane_id()) < D.k ? keys_in[static_cast<size_t>(li) * D.k + lane_id()] : kSentinel;
    ggm_seed_node<T, MET>(X, Xn, D, li, i, in, own_b ? 0 : nA, static_cast<uint64_t>(own_b ? nA : n_all - nA), level,
                          seed, G, reserved);
}

// Alg. 3 line 11: G[i] = k smallest unique keys of the refined list
// and the reserved half G^v.
__global__ void k_ggm_finalize(Dims D, Graph G, const uint64_t* __restrict__ reserved) {
    extern __shared__ uint64_t fin_scratch[];  // 32 u64 per warp
    const int64_t i = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (i >= D.n) return;
    const uint32_t lane = lane_id();
    const int k = D.k, kr = k - (k + 1) / 2;
    uint64_t cur = static_cast<int>(lane) < k ? G.keys[static_cast<size_t>(i) * k + lane] : kSentinel;
    uint32_t bits = 0;  // flags are not needed after the merge
    const uint64_t cand = static_cast<int>(lane) < kr ? reserved[static_cast<size_t>(i) * kr + lane] : kSentinel;
    warp_merge_list(cur, bits, cand, fin_scratch + (threadIdx.x >> 5) * 32);
    if (static_cast<int>(lane) < k) G.keys[static_cast<size_t>(i) * k + lane] = cur;
}

}  // namespace knng
