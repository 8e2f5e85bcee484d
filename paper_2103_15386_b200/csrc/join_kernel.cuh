// join_kernel.cuh -- the local join of Alg. 1.
//
// One CTA (128 threads) per node x with m = |G_new(x)| > 0.
//  gather : the m NEW and q OLD sample rows are staged into shared memory
//           with cp.async 16-B copies (L2-only .cg), slab by slab over the
//           dimensions (SLAB = 32 dims per stage, double-buffered), so any d
//           works with a fixed shared-memory footprint ("sub-vectors").
//  tile   : the CalculateDistances tile of P:181-194 as a register-blocked
//           contraction: each thread owns a 4x4 block of (NEW row, sample
//           column) pairs, lower-triangular blocks for NEW-NEW, all blocks
//           for NEW-OLD.  Every pair keeps one accumulator and walks the
//           dimensions in order, which is exactly the canonical distance of
//           D5/D6 -- results are bit-identical to the oracle's.
//  select : GetNearestObject (Alg. 2) as packed (dist, id) u64 minima: a
//           per-thread pre-reduction then shared-memory atomicMin -- the
//           paper's atomicMin on (v, d) with the (dist, id) order D3.
//  update : each selected candidate below its target's iteration-start k-th
//           key (an exact filter, D17) is appended to the target's bucket;
//           a full bucket falls back to the paper's locked insertion into
//           the list.  Buckets are merged by k_merge_sample.
#pragma once
#include <type_traits>

#include "graph_kernels.cuh"

namespace knng {

constexpr int kJoinThreads = 128;
constexpr int kMaxSlots = 64;  // m <= 32 NEW (padded to 4) + q <= 32 OLD

template <typename T>
struct SlabCfg;
template <>
struct SlabCfg<float> {
    static constexpr int kDims = 32;          // dims per stage
    static constexpr int kStride = 36;        // elements per smem row (pad 16 B)
    static constexpr int kChunkElems = 4;     // elements per 16-B chunk
};
template <>
struct SlabCfg<uint8_t> {
    static constexpr int kDims = 32;
    static constexpr int kStride = 48;
    static constexpr int kChunkElems = 16;
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
    const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ bool allowed_pair(int64_t boundary, uint32_t a, uint32_t b) {
    return boundary < 0 || ((static_cast<int64_t>(a) >= boundary) != (static_cast<int64_t>(b) >= boundary));
}

// InsertIntoNNList under the per-list spinlock: the overflow path
// of a full bucket.  Order-independent with the bucket merge (D17).
__device__ void locked_insert(Graph G, int k, uint32_t t, uint64_t key) {
    uint32_t* lk = G.lock + t;
    while (atomicCAS(lk, 0u, 1u) != 0u) __nanosleep(40);
    __threadfence();
    uint64_t* L = G.keys + static_cast<size_t>(t) * k;
    if (key < __ldcg(L + k - 1)) {
        bool dup = false;
        int below = 0;
        for (int j = 0; j < k; ++j) {
            const uint64_t lj = __ldcg(L + j);
            dup |= key_id(lj) == key_id(key);
            below += lj < key ? 1 : 0;
        }
        if (!dup) {
            for (int j = k - 1; j > below; --j) __stcg(L + j, __ldcg(L + j - 1));
            __stcg(L + below, key);
            const uint32_t m = __ldcg(G.newmask + t);
            const uint32_t lowm = (1u << below) - 1u;
            const uint32_t nm = ((m & lowm) | (1u << below) | ((m << 1) & ~(lowm | (1u << below)))) & kmask_of(k);
            __stcg(G.newmask + t, nm);
        }
    }
    __threadfence();
    atomicExch(lk, 0u);
}

__device__ __forceinline__ void emit_candidate(Graph G, int k, int B, uint32_t target, uint64_t key,
                                               unsigned int* c_cand, unsigned int* c_app, unsigned int* c_ovf) {
    if (key == kSentinel) return;  // D15
    atomicAdd(c_cand, 1u);
    if (!(key < __ldg(G.kth + target))) return;  // cannot enter (exact, D17)
    atomicAdd(c_app, 1u);
    const uint32_t slot = atomicAdd(G.bcnt + target, 1u);
    if (slot < static_cast<uint32_t>(B)) {
        G.bucket[static_cast<size_t>(target) * B + slot] = key;
    } else {
        atomicAdd(c_ovf, 1u);
        locked_insert(G, k, target, key);
    }
}

template <typename T, bool COS>
__global__ void __launch_bounds__(kJoinThreads)
k_join(const T* __restrict__ X, const float* __restrict__ Xn, Dims D, Graph G, Samples S,
       int64_t boundary, int aligned16, DevStats* __restrict__ stats) {
    using Cfg = SlabCfg<T>;
    using E = typename std::conditional<COS, float, T>::type;
    constexpr int SD = Cfg::kDims, RS = Cfg::kStride, CE = Cfg::kChunkElems;
    constexpr int CPR = SD / CE;  // 16-B chunks per row per stage
    const E* __restrict__ V = COS ? reinterpret_cast<const E*>(Xn) : reinterpret_cast<const E*>(X);

    __shared__ __align__(16) E rows[2][kMaxSlots * RS];
    __shared__ uint32_t ids[kMaxSlots];
    __shared__ unsigned long long mn_nn[32], mn_no[32], mn_on[32];
    __shared__ unsigned int c_pairs, c_cand, c_app, c_ovf;

    const int tid = threadIdx.x;
    const int d = D.d, cap = D.cap;
    const int nslab = (d + SD - 1) / SD;

    for (int64_t x = blockIdx.x; x < D.n; x += gridDim.x) {
        const int m = S.gcnt[2 * x], q = S.gcnt[2 * x + 1];
        if (m == 0) continue;  // no NEW sample: nothing to join (block-uniform)
        const int mpad = (m + 3) & ~3, qpad = (q + 3) & ~3;
        const int mg = mpad >> 2, qg = qpad >> 2;
        const int nslots = mpad + qpad;
        __syncthreads();  // previous node's smem fully consumed
        if (tid < kMaxSlots) {
            uint32_t id = 0xFFFFFFFFu;
            if (tid < m) id = S.G[static_cast<size_t>(x) * cap + tid];
            else if (tid >= mpad && tid - mpad < q)
                id = S.G[static_cast<size_t>(D.n) * cap + static_cast<size_t>(x) * cap + (tid - mpad)];
            ids[tid] = id;
        }
        if (tid < 32) {
            mn_nn[tid] = kSentinel;
            mn_no[tid] = kSentinel;
            mn_on[tid] = kSentinel;
        }
        if (tid == 0) { c_pairs = 0; c_cand = 0; c_app = 0; c_ovf = 0; }
        __syncthreads();

        // block assignment: NN lower-triangular blocks, then NO blocks
        const int nnn = mg * (mg + 1) / 2;
        const int nb = nnn + mg * qg;
        int I = 0, J = 0;
        const bool active = tid < nb;
        if (active) {
            if (tid < nnn) {
                I = static_cast<int>((sqrtf(8.0f * tid + 1.0f) - 1.0f) * 0.5f);
                while ((I + 1) * (I + 2) / 2 <= tid) ++I;
                while (I * (I + 1) / 2 > tid) --I;
                J = tid - I * (I + 1) / 2;
            } else {
                const int t2 = tid - nnn;
                I = t2 / qg;
                J = mg + t2 % qg;
            }
        }
        // column slot base: NN columns are NEW slots, NO columns start at mpad
        const int rbase = 4 * I;
        const int cbase = (J < mg) ? 4 * J : mpad + 4 * (J - mg);

        float acc[4][4];
        unsigned int iacc[4][4];
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
            for (int c = 0; c < 4; ++c) { acc[r][c] = 0.0f; iacc[r][c] = 0u; }

        auto issue = [&](int slab, int stage) {
            const int d0 = slab * SD;
            for (int c = tid; c < nslots * CPR; c += kJoinThreads) {
                const int slot = c / CPR, part = c - slot * CPR;
                const int e0 = d0 + part * CE;
                const uint32_t id = ids[slot];
                int cnt = 0;
                const E* src = V;
                if (id != 0xFFFFFFFFu && e0 < d) {
                    cnt = min(CE, d - e0);
                    src = V + static_cast<size_t>(id) * d + e0;
                }
                E* dst = &rows[stage][slot * RS + part * CE];
                if (aligned16) {
                    cp_async16(dst, src, cnt * static_cast<int>(sizeof(E)));
                } else {  // rows not 16-B aligned (d * sizeof(E) % 16 != 0)
#pragma unroll
                    for (int e = 0; e < CE; ++e) dst[e] = e < cnt ? __ldg(src + e) : E(0);
                }
            }
            cp_async_commit();
        };

        issue(0, 0);
        for (int sl = 0; sl < nslab; ++sl) {
            if (sl + 1 < nslab) {
                issue(sl + 1, (sl + 1) & 1);
                cp_async_wait<1>();
            } else {
                cp_async_wait<0>();
            }
            __syncthreads();
            if (active) {
                const E* R = rows[sl & 1];
                if constexpr (std::is_same<E, float>::value) {
#pragma unroll 2
                    for (int i = 0; i < SD; i += 4) {
                        float4 a[4], b[4];
#pragma unroll
                        for (int r = 0; r < 4; ++r) a[r] = *reinterpret_cast<const float4*>(R + (rbase + r) * RS + i);
#pragma unroll
                        for (int c = 0; c < 4; ++c) b[c] = *reinterpret_cast<const float4*>(R + (cbase + c) * RS + i);
#pragma unroll
                        for (int r = 0; r < 4; ++r)
#pragma unroll
                            for (int c = 0; c < 4; ++c) {
                                if constexpr (COS) {
                                    acc[r][c] = fmaf(a[r].x, b[c].x, acc[r][c]);
                                    acc[r][c] = fmaf(a[r].y, b[c].y, acc[r][c]);
                                    acc[r][c] = fmaf(a[r].z, b[c].z, acc[r][c]);
                                    acc[r][c] = fmaf(a[r].w, b[c].w, acc[r][c]);
                                } else {
                                    float t;
                                    t = a[r].x - b[c].x; acc[r][c] = fmaf(t, t, acc[r][c]);
                                    t = a[r].y - b[c].y; acc[r][c] = fmaf(t, t, acc[r][c]);
                                    t = a[r].z - b[c].z; acc[r][c] = fmaf(t, t, acc[r][c]);
                                    t = a[r].w - b[c].w; acc[r][c] = fmaf(t, t, acc[r][c]);
                                }
                            }
                    }
                } else {
                    // uint8: exact integer sum of squares (D5), 4 dims per step
#pragma unroll 2
                    for (int i = 0; i < SD; i += 4) {
                        uint32_t a[4], b[4];
#pragma unroll
                        for (int r = 0; r < 4; ++r) a[r] = *reinterpret_cast<const uint32_t*>(R + (rbase + r) * RS + i);
#pragma unroll
                        for (int c = 0; c < 4; ++c) b[c] = *reinterpret_cast<const uint32_t*>(R + (cbase + c) * RS + i);
#pragma unroll
                        for (int r = 0; r < 4; ++r)
#pragma unroll
                            for (int c = 0; c < 4; ++c) {
                                const uint32_t ad = __vabsdiffu4(a[r], b[c]);
                                iacc[r][c] = __dp4a(ad, ad, iacc[r][c]);
                            }
                    }
                }
            }
            __syncthreads();
        }

        // ---- selection (Alg. 2): per-thread pre-reduction + smem atomicMin
        if (active) {
            const bool nn = J < mg;
            unsigned pairs = 0;
            uint64_t colbest[4] = {kSentinel, kSentinel, kSentinel, kSentinel};
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const int u = rbase + r;
                uint64_t rowbest = kSentinel;
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const int w = cbase + c;
                    bool valid;
                    if (nn) valid = u < m && w < u;
                    else valid = u < m && (w - mpad) < q;
                    if (valid) valid = allowed_pair(boundary, ids[u], ids[w]);
                    if (!valid) continue;
                    float dist;
                    if constexpr (COS) {
                        const float rr = 1.0f - acc[r][c];
                        dist = rr > 0.0f ? rr : 0.0f;
                    } else if constexpr (std::is_same<E, float>::value) {
                        dist = acc[r][c];
                    } else {
                        dist = static_cast<float>(iacc[r][c]);
                    }
                    ++pairs;
                    const uint64_t kr = make_key(dist, ids[w]);
                    const uint64_t kc = make_key(dist, ids[u]);
                    rowbest = kr < rowbest ? kr : rowbest;
                    colbest[c] = kc < colbest[c] ? kc : colbest[c];
                }
                if (rowbest != kSentinel) {
                    if (nn) atomicMin(&mn_nn[u], static_cast<unsigned long long>(rowbest));
                    else atomicMin(&mn_no[u], static_cast<unsigned long long>(rowbest));
                }
            }
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                if (colbest[c] == kSentinel) continue;
                const int w = cbase + c;
                if (nn) atomicMin(&mn_nn[w], static_cast<unsigned long long>(colbest[c]));
                else atomicMin(&mn_on[w - mpad], static_cast<unsigned long long>(colbest[c]));
            }
            if (pairs) atomicAdd(&c_pairs, pairs);
        }
        __syncthreads();

        // ---- update: NEW sample u gets nearest other NEW and nearest OLD
        // (Alg. 1 lines 12-25); OLD sample gets nearest NEW (lines 26-31).
        if (tid < m) {
            const uint32_t u = ids[tid];
            emit_candidate(G, D.k, D.B, u, mn_nn[tid], &c_cand, &c_app, &c_ovf);
            emit_candidate(G, D.k, D.B, u, mn_no[tid], &c_cand, &c_app, &c_ovf);
        }
        if (tid >= 32 && tid - 32 < q) {
            const int j = tid - 32;
            emit_candidate(G, D.k, D.B, ids[mpad + j], mn_on[j], &c_cand, &c_app, &c_ovf);
        }
        __syncthreads();
        if (tid == 0) {
            atomicAdd(&stats->joins, 1ull);
            atomicAdd(&stats->sum_m, static_cast<unsigned long long>(m));
            atomicAdd(&stats->sum_q, static_cast<unsigned long long>(q));
            atomicAdd(&stats->rows, static_cast<unsigned long long>(m + q));
            atomicAdd(&stats->dist_evals, static_cast<unsigned long long>(c_pairs));
            atomicAdd(&stats->candidates, static_cast<unsigned long long>(c_cand));
            atomicAdd(&stats->appended, static_cast<unsigned long long>(c_app));
            if (c_ovf) atomicAdd(&stats->overflow, static_cast<unsigned long long>(c_ovf));
        }
    }
}

}  // namespace knng
