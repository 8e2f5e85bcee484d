// join_locked.cuh -- the paper's own update design, kept for the ablation of
// one thread block per object,
// the NEW-NEW pairs mapped to threads by Eq. 1-2, and the
// selected (or, for GNND-r1, all) neighbour pairs inserted IMMEDIATELY into
// the k-NN lists under spinlocks instead of the bulk-synchronous
// lock-free buckets of the default path (D17, D34).
//
//   update mode 1 "full"     GNND-r1: every produced pair offered to
//                            its list -- per sample u, all distances to it are
//                            sorted (bitonic) and merged with G[u]
//   update mode 2 "locked"   GNND (P:199 + P:244): the nearest objects of
//                            Alg. 2 only, one spinlock per list segment
//                            ("multiple spinlocks")
//   update mode 3 "locked1"  GNND-r2: as 2 with one lock per whole list
//
// Every mode gives the oracle's lists: a bounded sorted list fed any order of
// offers ends as the smallest unique keys of the union (D17; per segment for
// segmented lists, D40), and keys are canonical per (target, id) (D5).
#pragma once
#include "join_ws.cuh"

namespace knng {

constexpr int kLkThreads = 128;
constexpr int kLkRows = 64;   // m + q <= 2 cap <= 64 sample rows
constexpr int kLkDims = 64;   // dimensions staged per pass

// one dimension of the canonical accumulation (D5, D6, D39)
template <int MET>
__device__ __forceinline__ float lk_acc(float x, float y, float acc) {
    if constexpr (MET == kMetCos) return fmaf(x, y, acc);
    if constexpr (MET == kMetChi2) return chi2_term(x, y, acc);
    const float t = x - y;
    return fmaf(t, t, acc);
}

// Immediate insert of up to 64 offers (two 32-key chunks held one per lane)
// into list t under its lock (segment locks: one per segment, the offers
// routed by id % s).  bits: bit0 NEW, bit1 entered during this iteration
// (accepted count, read back by k_merge_sample).
__device__ __forceinline__ void lk_acquire(unsigned int* lk) {
    if (lane_id() == 0) {
        unsigned int ns = 8;
        while (atomicCAS(lk, 0u, 1u) != 0u) {
            __nanosleep(ns);
            ns = ns < 256 ? 2 * ns : 256;
        }
    }
    __syncwarp();
    __threadfence();
}
__device__ __forceinline__ void lk_release(unsigned int* lk) {
    __threadfence();
    __syncwarp();
    if (lane_id() == 0) atomicExch(lk, 0u);
}

__device__ __forceinline__ void lk_insert(Graph& G, const Dims& D, int64_t t, uint64_t c0, uint64_t c1,
                                          uint64_t* scratch, bool one_lock) {
    const uint32_t lane = lane_id();
    const int s = D.k > 32 ? D.k / 32 : 1;  // segments (D40)
    const int per = D.k / s;
    if (one_lock) lk_acquire(G.lock + t * s);
    for (int g = 0; g < s; ++g) {
        uint64_t a = c0, b = c1;
        if (s > 1) {
            a = (a != kSentinel && key_id(a) % s == static_cast<uint32_t>(g)) ? a : kSentinel;
            b = (b != kSentinel && key_id(b) % s == static_cast<uint32_t>(g)) ? b : kSentinel;
        }
        if (!__any_sync(kFull, a != kSentinel || b != kSentinel)) continue;
        if (!one_lock) lk_acquire(G.lock + t * s + g);
        // segment g of list t: entries [g * 32, g * 32 + per) (segment-major)
        uint64_t* L = G.keys + static_cast<size_t>(t) * D.k + static_cast<size_t>(g) * 32;
        const bool in = static_cast<int>(lane) < per;
        uint64_t cur = in ? __ldcg(L + lane) : kSentinel;
        const uint32_t nm = __ldcg(G.newmask + t * s + g), im = __ldcg(G.imask + t * s + g);
        uint32_t bits = in ? (((nm >> lane) & 1u) | (((im >> lane) & 1u) << 1)) : 0u;
        warp_merge_list(cur, bits, a, scratch);
        if (__any_sync(kFull, b != kSentinel)) warp_merge_list(cur, bits, b, scratch);
        if (!in) {
            cur = kSentinel;
            bits = 0;
        }
        if (in) __stcg(L + lane, cur);
        const uint32_t nm2 = __ballot_sync(kFull, in && (bits & 1u));
        const uint32_t im2 = __ballot_sync(kFull, in && (bits & 2u));
        if (lane == 0) {
            __stcg(G.newmask + t * s + g, nm2);
            __stcg(G.imask + t * s + g, im2);
        }
        if (!one_lock) lk_release(G.lock + t * s + g);
    }
    if (one_lock) lk_release(G.lock + t * s);
}

template <typename T, int MET, bool FULL>
__global__ void __launch_bounds__(kLkThreads)
k_join_locked(const T* __restrict__ X, const float* __restrict__ Xn, Dims D, Graph G, Samples S, int64_t boundary,
              int one_lock, DevStats* __restrict__ stats) {
    using E = typename std::conditional<MET == kMetCos, float, T>::type;
    constexpr bool kInt = std::is_same<E, uint8_t>::value;  // exact integer L2 (D5)
    using Acc = typename std::conditional<kInt, int, float>::type;
    const E* __restrict__ V = MET == kMetCos ? reinterpret_cast<const E*>(Xn) : reinterpret_cast<const E*>(X);
    __shared__ uint32_t ids[kLkRows];
    __shared__ E rows[kLkRows][kLkDims + (kInt ? 4 : 1)];
    __shared__ float dist[kLkRows * (kLkRows - 1) / 2 + kLkRows * kLkRows / 4 + 32];
    __shared__ uint64_t scratch[kLkThreads / 32][32];
    constexpr int kMaxPairsPerThread = (32 * 31 / 2 + 32 * 32 + kLkThreads - 1) / kLkThreads;
    const int tid = threadIdx.x, warp = tid >> 5;
    const uint32_t lane = lane_id();
    const bool restricted = boundary >= 0;
    unsigned long long n_pairs = 0, n_cand = 0;

    for (int64_t x = blockIdx.x; x < D.n; x += gridDim.x) {
        const int m = S.gcnt[2 * x], q = S.gcnt[2 * x + 1];
        if (m == 0) continue;  // no NEW sample: no join (block-uniform)
        if (tid < m) ids[tid] = S.G[static_cast<size_t>(x) * D.cap + tid];
        else if (tid < m + q) ids[tid] = S.G[static_cast<size_t>(D.n) * D.cap + static_cast<size_t>(x) * D.cap + tid - m];
        __syncthreads();
        const int nnn = m * (m - 1) / 2, npairs = nnn + m * q;
        // ---- CalculateDistances (Alg. 1 lines 11, 19): thread t owns pairs
        // t, t + 128, ...; NEW-NEW pair t is (u, v) of Eq. 1-2,
        // stored at D_new[u (u-1)/2 + v]; NEW-OLD pair (u, j) at nnn + u q + j
        Acc acc[kMaxPairsPerThread];
        int pa[kMaxPairsPerThread], pb[kMaxPairsPerThread];
#pragma unroll
        for (int r = 0; r < kMaxPairsPerThread; ++r) {
            acc[r] = Acc(0);
            const int t = tid + r * kLkThreads;
            pa[r] = -1;
            pb[r] = -1;
            if (t < nnn) {
                int u = static_cast<int>(ceilf(sqrtf(2.0f * t + 2.25f) - 0.5f));
                // exact integer correction of the float evaluation
                while (u * (u - 1) / 2 > t) --u;
                while ((u + 1) * u / 2 <= t) ++u;
                pa[r] = u;
                pb[r] = t - u * (u - 1) / 2;
            } else if (t < npairs) {
                const int o = t - nnn;
                pa[r] = o / q;
                pb[r] = m + o % q;
            }
        }
        for (int d0 = 0; d0 < D.d; d0 += kLkDims) {
            const int dw = min(kLkDims, D.d - d0);
            __syncthreads();
            for (int e = tid; e < (m + q) * dw; e += kLkThreads) {
                const int r = e / dw, c = e - r * dw;
                rows[r][c] = V[static_cast<size_t>(ids[r]) * D.d + d0 + c];
            }
            __syncthreads();
#pragma unroll
            for (int r = 0; r < kMaxPairsPerThread; ++r) {
                if (pa[r] < 0) continue;
                const E* ra = rows[pa[r]];
                const E* rb = rows[pb[r]];
                for (int c = 0; c < dw; ++c) {
                    if constexpr (kInt) {
                        const int t = static_cast<int>(ra[c]) - static_cast<int>(rb[c]);
                        acc[r] += t * t;
                    } else {
                        acc[r] = lk_acc<MET>(static_cast<float>(ra[c]), static_cast<float>(rb[c]), acc[r]);
                    }
                }
            }
        }
#pragma unroll
        for (int r = 0; r < kMaxPairsPerThread; ++r) {
            const int t = tid + r * kLkThreads;
            if (pa[r] < 0) continue;
            float dd;
            if constexpr (MET == kMetCos) {
                const float x1 = 1.0f - acc[r];
                dd = x1 > 0.0f ? x1 : 0.0f;
            } else {
                dd = static_cast<float>(acc[r]);
            }
            const bool ok = !restricted || allowed_pair(boundary, ids[pa[r]], ids[pb[r]]);
            dist[t] = ok ? dd : __int_as_float(-1);  // -NaN marks a skipped pair (D22)
            n_pairs += ok;
        }
        __syncthreads();
        // ---- selection + immediate update: warp w takes targets w, w+4, ...
        auto dnn = [&](int u, int w) { return u > w ? dist[u * (u - 1) / 2 + w] : dist[w * (w - 1) / 2 + u]; };
        for (int tg = warp; tg < m + q; tg += kLkThreads / 32) {
            // offers to target tg: NEW u -> other NEW (lane j) + OLD (lane j);
            // OLD w -> NEW (lane j).  Keys (d, id); skipped pairs: none.
            uint64_t o0 = kSentinel, o1 = kSentinel;
            if (tg < m) {
                const int j = static_cast<int>(lane);
                if (j < m && j != tg) {
                    const float dd = dnn(tg, j);
                    if (!(__float_as_int(dd) == -1)) o0 = make_key(dd, ids[j]);
                }
                if (j < q) {
                    const float dd = dist[nnn + tg * q + j];
                    if (!(__float_as_int(dd) == -1)) o1 = make_key(dd, ids[m + j]);
                }
            } else {
                const int j = static_cast<int>(lane), w = tg - m;
                if (j < m) {
                    const float dd = dist[nnn + j * q + w];
                    if (!(__float_as_int(dd) == -1)) o0 = make_key(dd, ids[j]);
                }
            }
            if constexpr (!FULL) {
                // Alg. 2 (GetNearestObject): the minimum of each offer set
                uint64_t m0 = o0, m1 = o1;
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) {
                    const uint64_t a = shfl_xor_u64(m0, off), b = shfl_xor_u64(m1, off);
                    m0 = a < m0 ? a : m0;
                    m1 = b < m1 ? b : m1;
                }
                o0 = lane == 0 ? m0 : kSentinel;
                o1 = lane == 0 ? m1 : kSentinel;
            }
            n_cand += __popc(__ballot_sync(kFull, o0 != kSentinel)) + __popc(__ballot_sync(kFull, o1 != kSentinel));
            if (__any_sync(kFull, o0 != kSentinel || o1 != kSentinel))
                lk_insert(G, D, ids[tg], o0, o1, scratch[warp], one_lock != 0);
        }
        __syncthreads();
    }
    __shared__ unsigned long long red[2];
    if (tid == 0) red[0] = red[1] = 0;
    __syncthreads();
    if (lane == 0) {
        atomicAdd(&red[1], n_cand);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) n_pairs += __shfl_xor_sync(kFull, n_pairs, o);
    if (lane == 0) atomicAdd(&red[0], n_pairs);
    __syncthreads();
    if (tid == 0) {
        if (red[0]) atomicAdd(&stats->dist_evals, red[0]);
        if (red[1]) atomicAdd(&stats->candidates, red[1]);
    }
}

}  // namespace knng
