// join_kernel.cuh -- the local join of Alg. 1.
//
// k_join: one CTA (128 threads) per node x with m = |G_new(x)| > 0,
// persistent over nodes.
//  gather : the m NEW and q OLD sample rows are staged into shared memory
//           with cp.async 16-B copies (L2-only .cg), slab by slab over the
//           dimensions (32 dims per stage, double-buffered), so any d works
//           with a fixed shared-memory footprint ("sub-vectors").
//  tile   : the CalculateDistances tile of P:181-194 as a register-blocked
//           contraction: each thread owns a 4x4 block of (NEW row, sample
//           column) pairs, lower-triangular blocks for NEW-NEW, all blocks
//           for NEW-OLD.  Every pair keeps one accumulator and walks the
//           dimensions in order: exactly the canonical distance of D5/D6, so
//           results are bit-identical to the oracle's.
//  select : GetNearestObject (Alg. 2) as packed (dist, id) u64 minima: a
//           per-thread pre-reduction then shared-memory atomicMin -- the
//           paper's atomicMin on (v, d) with the (dist, id) order D3.
//  output : the 2m + q selected keys go to a fixed per-node slot range of
//           S.cand (coalesced, no atomics); k_cand_scatter files them.
//
// k_cand_scatter: one thread per candidate slot: drops keys that cannot
// enter (>= the target's iteration-start k-th key: exact, D17) and appends
// the rest to the target's CSR bucket (never overflows, see k_scan_*).
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

template <typename T, bool COS>
__global__ void __launch_bounds__(kJoinThreads)
k_join(const T* __restrict__ X, const float* __restrict__ Xn, Dims D, Samples S, int64_t boundary,
       int aligned16, DevStats* __restrict__ stats) {
    using Cfg = SlabCfg<T>;
    using E = typename std::conditional<COS, float, T>::type;
    constexpr int SD = Cfg::kDims, RS = Cfg::kStride, CE = Cfg::kChunkElems;
    constexpr int CPR = SD / CE;  // 16-B chunks per row per stage
    const E* __restrict__ V = COS ? reinterpret_cast<const E*>(Xn) : reinterpret_cast<const E*>(X);

    __shared__ __align__(16) E rows[2][kMaxSlots * RS];
    __shared__ uint32_t ids[kMaxSlots];
    __shared__ unsigned long long mn_nn[32], mn_no[32], mn_on[32];
    __shared__ unsigned int c_pairs;

    const int tid = threadIdx.x;
    const int d = D.d, cap = D.cap;
    const int nslab = (d + SD - 1) / SD;
    unsigned long long my_joins = 0, my_m = 0, my_q = 0;

    for (int64_t x = blockIdx.x; x < D.n; x += gridDim.x) {
        const int m = S.gcnt[2 * x], q = S.gcnt[2 * x + 1];
        if (m == 0) continue;  // no NEW sample: nothing to join (block-uniform)
        const int mpad = (m + 3) & ~3, qpad = (q + 3) & ~3;
        const int mg = mpad >> 2, qg = qpad >> 2;
        const int nslots = mpad + qpad;
        __syncthreads();  // previous node's shared memory fully consumed
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
        if (tid == 0) c_pairs = 0;
        __syncthreads();

        // block assignment: NN lower-triangular blocks (I >= J), then NO blocks
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
        const bool nn = J < mg;
        const int rbase = 4 * I;
        const int cbase = nn ? 4 * J : mpad + 4 * (J - mg);
        const int aoff = rbase * RS, boff = cbase * RS;

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
                const E* __restrict__ A = rows[sl & 1] + aoff;
                const E* __restrict__ B = rows[sl & 1] + boff;
                if constexpr (std::is_same<E, float>::value) {
#pragma unroll
                    for (int i = 0; i < SD; i += 4) {
                        float4 a[4], b[4];
#pragma unroll
                        for (int r = 0; r < 4; ++r) a[r] = *reinterpret_cast<const float4*>(A + r * RS + i);
#pragma unroll
                        for (int c = 0; c < 4; ++c) b[c] = *reinterpret_cast<const float4*>(B + c * RS + i);
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
#pragma unroll
                    for (int i = 0; i < SD; i += 4) {
                        uint32_t a[4], b[4];
#pragma unroll
                        for (int r = 0; r < 4; ++r) a[r] = *reinterpret_cast<const uint32_t*>(A + r * RS + i);
#pragma unroll
                        for (int c = 0; c < 4; ++c) b[c] = *reinterpret_cast<const uint32_t*>(B + c * RS + i);
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
            unsigned pairs = 0;
            uint64_t colbest[4] = {kSentinel, kSentinel, kSentinel, kSentinel};
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const int u = rbase + r;
                uint64_t rowbest = kSentinel;
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const int w = cbase + c;
                    bool valid = nn ? (u < m && w < u) : (u < m && (w - mpad) < q);
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

        // ---- output: slot j of node x holds c_nn(u_j) (j < m), c_no(u_j)
        // (m <= j < 2m), c_on(w_j) (2m <= j < 2m + q)  (Alg. 1 lines 12-31)
        uint64_t* out = S.cand + static_cast<size_t>(x) * (3 * cap);
        const int total = 2 * m + q;
        for (int j = tid; j < total; j += kJoinThreads) {
            uint64_t v;
            if (j < m) v = mn_nn[j];
            else if (j < 2 * m) v = mn_no[j - m];
            else v = mn_on[j - 2 * m];
            out[j] = v;
        }
        if (tid == 0) {
            ++my_joins;
            my_m += static_cast<unsigned long long>(m);
            my_q += static_cast<unsigned long long>(q);
            atomicAdd(&stats->dist_evals, static_cast<unsigned long long>(c_pairs));
        }
    }
    if (tid == 0 && my_joins) {
        atomicAdd(&stats->joins, my_joins);
        atomicAdd(&stats->sum_m, my_m);
        atomicAdd(&stats->sum_q, my_q);
        atomicAdd(&stats->rows, my_m + my_q);
    }
}

// File the join outputs into the targets' buckets.  Slot j of node x: its
// target is G_new(x)[j] (j < 2m, as c_nn / c_no of that NEW sample) or
// G_old(x)[j - 2m].
__global__ void k_cand_scatter(Dims D, Graph G, Samples S, DevStats* __restrict__ stats) {
    __shared__ unsigned int c_cand, c_app;
    if (threadIdx.x == 0) { c_cand = 0; c_app = 0; }
    __syncthreads();
    const int slots = 3 * D.cap;
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < D.n * slots) {
        const int64_t x = i / slots;
        const int j = static_cast<int>(i - x * slots);
        const int m = S.gcnt[2 * x], q = S.gcnt[2 * x + 1];
        if (m > 0 && j < 2 * m + q) {
            const uint64_t key = S.cand[i];
            if (key != kSentinel) {  // D15: the (inf, inf) tuple inserts nothing
                atomicAdd(&c_cand, 1u);
                const uint32_t t = j < 2 * m
                    ? S.G[static_cast<size_t>(x) * D.cap + (j < m ? j : j - m)]
                    : S.G[static_cast<size_t>(D.n) * D.cap + static_cast<size_t>(x) * D.cap + (j - 2 * m)];
                if (key < G.kth[t]) {  // else it cannot enter G[t] (exact, D17)
                    atomicAdd(&c_app, 1u);
                    const uint32_t slot = atomicAdd(G.bcnt + t, 1u);
                    G.bucket[G.boff[t] + slot] = key;
                }
            }
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        if (c_cand) atomicAdd(&stats->candidates, static_cast<unsigned long long>(c_cand));
        if (c_app) atomicAdd(&stats->appended, static_cast<unsigned long long>(c_app));
    }
}

}  // namespace knng
