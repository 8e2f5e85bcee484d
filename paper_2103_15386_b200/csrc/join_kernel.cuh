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

constexpr int kJoinNodes = 4;  // nodes per CTA batch
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
    static constexpr int kDims = 128;         // 128-B row slab, like f32
    static constexpr int kStride = 144;
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

// One CTA handles a batch of NB consecutive nodes per step of a persistent
// loop; the 4x4 register blocks of all NB tiles form one flat list spread
// over the CTA's 64 NB threads, so warps stay full even though a single
// node's tile has only ~35-100 blocks (the one-node-per-CTA layout left
// ~40% of the FP lanes idle).
template <typename T, int MET, int NB>
__global__ void __launch_bounds__(NB * 64, 2)
k_join(const T* __restrict__ X, const float* __restrict__ Xn, Dims D, Samples S, int64_t boundary,
       int aligned16, DevStats* __restrict__ stats) {
    using Cfg = SlabCfg<T>;
    using E = typename std::conditional<MET == kMetCos, float, T>::type;
    constexpr bool kFloat = std::is_same<E, float>::value;
    using Acc = typename std::conditional<kFloat, float, unsigned int>::type;
    constexpr int SD = Cfg::kDims, RS = Cfg::kStride, CE = Cfg::kChunkElems;
    constexpr int CPR = SD / CE;               // 16-B chunks per row per stage
    constexpr int THREADS = NB * 64;
    constexpr int TILE = kMaxSlots * RS;       // elements of one node's stage
    constexpr int ROUNDS = (NB * 100 + THREADS - 1) / THREADS;  // <= 100 blocks per node
    const E* __restrict__ V = MET == kMetCos ? reinterpret_cast<const E*>(Xn) : reinterpret_cast<const E*>(X);

    extern __shared__ __align__(16) unsigned char join_smem[];
    E* rows = reinterpret_cast<E*>(join_smem);  // [2][NB][TILE]
    __shared__ uint32_t ids[NB][kMaxSlots];
    __shared__ unsigned long long mins[NB][3][32];  // c_nn, c_no (per NEW u), c_on (per OLD w)
    __shared__ int sm_m[NB], sm_q[NB], blk_pre[NB + 1], chk_pre[NB + 1];
    __shared__ unsigned int c_pairs;

    const int tid = threadIdx.x;
    const int d = D.d, cap = D.cap;
    const int nslab = (d + SD - 1) / SD;
    unsigned long long my_joins = 0, my_m = 0, my_q = 0;

    for (int64_t b0 = static_cast<int64_t>(blockIdx.x) * NB; b0 < D.n; b0 += static_cast<int64_t>(gridDim.x) * NB) {
        __syncthreads();  // previous batch fully consumed
        if (tid < NB) {
            const int64_t x = b0 + tid;
            int m = 0, q = 0;
            if (x < D.n) { m = S.gcnt[2 * x]; q = S.gcnt[2 * x + 1]; }
            if (m == 0) q = 0;  // no NEW sample: nothing to join
            sm_m[tid] = m;
            sm_q[tid] = q;
        }
        for (int i = tid; i < NB * 96; i += THREADS) (&mins[0][0][0])[i] = kSentinel;
        if (tid == 0) c_pairs = 0;
        __syncthreads();
        if (tid == 0) {
            int bp = 0, cp = 0;
            for (int i = 0; i < NB; ++i) {
                blk_pre[i] = bp;
                chk_pre[i] = cp;
                const int mg = (sm_m[i] + 3) >> 2, qg = (sm_q[i] + 3) >> 2;
                bp += mg * (mg + 1) / 2 + mg * qg;
                cp += 4 * (mg + qg) * CPR;
            }
            blk_pre[NB] = bp;
            chk_pre[NB] = cp;
        }
        for (int i = tid; i < NB * kMaxSlots; i += THREADS) {
            const int nd = i / kMaxSlots, slot = i - nd * kMaxSlots;
            const int m = sm_m[nd], q = sm_q[nd], mpad = (m + 3) & ~3;
            const int64_t x = b0 + nd;
            uint32_t id = 0xFFFFFFFFu;
            if (slot < m) id = S.G[static_cast<size_t>(x) * cap + slot];
            else if (slot >= mpad && slot - mpad < q)
                id = S.G[static_cast<size_t>(D.n) * cap + static_cast<size_t>(x) * cap + (slot - mpad)];
            ids[nd][slot] = id;
        }
        __syncthreads();
        const int total_blocks = blk_pre[NB];
        if (total_blocks == 0) continue;  // block-uniform
        const int total_chunks = chk_pre[NB];

        // this thread's blocks: (node, row base, col base, NN?) per round
        int b_node[ROUNDS], b_abase[ROUNDS], b_bbase[ROUNDS], b_rb[ROUNDS], b_cb[ROUNDS];
        bool b_nn[ROUNDS], b_on[ROUNDS];
#pragma unroll
        for (int r = 0; r < ROUNDS; ++r) {
            const int f = tid + r * THREADS;
            b_on[r] = f < total_blocks;
            int nd = 0;
            while (nd + 1 < NB && blk_pre[nd + 1] <= f) ++nd;
            const int t = f - blk_pre[nd];
            const int m = sm_m[nd], q = sm_q[nd];
            const int mpad = (m + 3) & ~3, mg = mpad >> 2, qg = (q + 3) >> 2;
            const int nnn = mg * (mg + 1) / 2;
            int I = 0, J = 0;
            if (b_on[r]) {
                if (t < nnn) {
                    I = static_cast<int>((sqrtf(8.0f * t + 1.0f) - 1.0f) * 0.5f);
                    while ((I + 1) * (I + 2) / 2 <= t) ++I;
                    while (I * (I + 1) / 2 > t) --I;
                    J = t - I * (I + 1) / 2;
                } else {
                    const int t2 = t - nnn;
                    I = t2 / qg;
                    J = mg + t2 % qg;
                }
            }
            b_node[r] = nd;
            b_nn[r] = J < mg;
            b_rb[r] = 4 * I;
            b_cb[r] = b_nn[r] ? 4 * J : mpad + 4 * (J - mg);
            b_abase[r] = nd * TILE + b_rb[r] * RS;
            b_bbase[r] = nd * TILE + b_cb[r] * RS;
        }

        Acc acc[ROUNDS][4][4];
#pragma unroll
        for (int r = 0; r < ROUNDS; ++r)
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int c = 0; c < 4; ++c) acc[r][i][c] = Acc(0);

        auto issue = [&](int slab, int stage) {
            const int d0 = slab * SD;
            E* base = rows + stage * NB * TILE;
            for (int c = tid; c < total_chunks; c += THREADS) {
                int nd = 0;
                while (nd + 1 < NB && chk_pre[nd + 1] <= c) ++nd;
                const int cl = c - chk_pre[nd];
                const int slot = cl / CPR, part = cl - slot * CPR;
                const int e0 = d0 + part * CE;
                const uint32_t id = ids[nd][slot];
                int cnt = 0;
                const E* src = V;
                if (id != 0xFFFFFFFFu && e0 < d) {
                    cnt = min(CE, d - e0);
                    src = V + static_cast<size_t>(id) * d + e0;
                }
                E* dst = base + nd * TILE + slot * RS + part * CE;
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
            const E* st = rows + (sl & 1) * NB * TILE;
#pragma unroll
            for (int r = 0; r < ROUNDS; ++r) {
                if (!b_on[r]) continue;
                const E* __restrict__ A = st + b_abase[r];
                const E* __restrict__ B = st + b_bbase[r];
                if constexpr (kFloat) {
#pragma unroll
                    for (int i = 0; i < SD; i += 4) {
                        float4 a[4], b[4];
#pragma unroll
                        for (int rr = 0; rr < 4; ++rr) a[rr] = *reinterpret_cast<const float4*>(A + rr * RS + i);
#pragma unroll
                        for (int c = 0; c < 4; ++c) b[c] = *reinterpret_cast<const float4*>(B + c * RS + i);
#pragma unroll
                        for (int rr = 0; rr < 4; ++rr)
#pragma unroll
                            for (int c = 0; c < 4; ++c) {
                                if constexpr (MET == kMetCos) {
                                    acc[r][rr][c] = fmaf(a[rr].x, b[c].x, acc[r][rr][c]);
                                    acc[r][rr][c] = fmaf(a[rr].y, b[c].y, acc[r][rr][c]);
                                    acc[r][rr][c] = fmaf(a[rr].z, b[c].z, acc[r][rr][c]);
                                    acc[r][rr][c] = fmaf(a[rr].w, b[c].w, acc[r][rr][c]);
                                } else if constexpr (MET == kMetChi2) {
                                    acc[r][rr][c] = chi2_term(a[rr].x, b[c].x, acc[r][rr][c]);
                                    acc[r][rr][c] = chi2_term(a[rr].y, b[c].y, acc[r][rr][c]);
                                    acc[r][rr][c] = chi2_term(a[rr].z, b[c].z, acc[r][rr][c]);
                                    acc[r][rr][c] = chi2_term(a[rr].w, b[c].w, acc[r][rr][c]);
                                } else {
                                    float t;
                                    t = a[rr].x - b[c].x; acc[r][rr][c] = fmaf(t, t, acc[r][rr][c]);
                                    t = a[rr].y - b[c].y; acc[r][rr][c] = fmaf(t, t, acc[r][rr][c]);
                                    t = a[rr].z - b[c].z; acc[r][rr][c] = fmaf(t, t, acc[r][rr][c]);
                                    t = a[rr].w - b[c].w; acc[r][rr][c] = fmaf(t, t, acc[r][rr][c]);
                                }
                            }
                    }
                } else {
                    // uint8: exact integer sum of squares (D5), 4 dims per step
#pragma unroll
                    for (int i = 0; i < SD; i += 4) {
                        uint32_t a[4], b[4];
#pragma unroll
                        for (int rr = 0; rr < 4; ++rr) a[rr] = *reinterpret_cast<const uint32_t*>(A + rr * RS + i);
#pragma unroll
                        for (int c = 0; c < 4; ++c) b[c] = *reinterpret_cast<const uint32_t*>(B + c * RS + i);
#pragma unroll
                        for (int rr = 0; rr < 4; ++rr)
#pragma unroll
                            for (int c = 0; c < 4; ++c) {
                                const uint32_t ad = __vabsdiffu4(a[rr], b[c]);
                                acc[r][rr][c] = __dp4a(ad, ad, acc[r][rr][c]);
                            }
                    }
                }
            }
            __syncthreads();
        }

        // ---- selection (Alg. 2): per-thread pre-reduction + smem atomicMin
        unsigned pairs = 0;
#pragma unroll
        for (int r = 0; r < ROUNDS; ++r) {
            if (!b_on[r]) continue;
            const int nd = b_node[r];
            const int m = sm_m[nd], q = sm_q[nd], mpad = (m + 3) & ~3;
            const bool nn = b_nn[r];
            const uint32_t* nid = ids[nd];
            unsigned long long* mn_nn = mins[nd][0];
            unsigned long long* mn_no = mins[nd][1];
            unsigned long long* mn_on = mins[nd][2];
            uint64_t colbest[4] = {kSentinel, kSentinel, kSentinel, kSentinel};
#pragma unroll
            for (int rr = 0; rr < 4; ++rr) {
                const int u = b_rb[r] + rr;
                uint64_t rowbest = kSentinel;
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const int w = b_cb[r] + c;
                    bool valid = nn ? (u < m && w < u) : (u < m && (w - mpad) < q);
                    if (valid) valid = allowed_pair(boundary, nid[u], nid[w]);
                    if (!valid) continue;
                    float dist;
                    if constexpr (MET == kMetCos) {
                        const float x1 = 1.0f - acc[r][rr][c];
                        dist = x1 > 0.0f ? x1 : 0.0f;
                    } else if constexpr (kFloat) {
                        dist = acc[r][rr][c];
                    } else {
                        dist = static_cast<float>(acc[r][rr][c]);
                    }
                    ++pairs;
                    const uint64_t kr = make_key(dist, nid[w]);
                    const uint64_t kc = make_key(dist, nid[u]);
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
                const int w = b_cb[r] + c;
                if (nn) atomicMin(&mn_nn[w], static_cast<unsigned long long>(colbest[c]));
                else atomicMin(&mn_on[w - mpad], static_cast<unsigned long long>(colbest[c]));
            }
        }
        if (pairs) atomicAdd(&c_pairs, pairs);
        __syncthreads();

        // ---- output: slot j of node x holds c_nn(u_j) (j < m), c_no(u_j)
        // (m <= j < 2m), c_on(w_j) (2m <= j < 2m + q)  (Alg. 1 lines 12-31)
        for (int i = tid; i < NB * 3 * 32; i += THREADS) {
            const int nd = i / 96, j = i - nd * 96;
            const int m = sm_m[nd], q = sm_q[nd];
            if (j >= 2 * m + q) continue;
            uint64_t v;
            if (j < m) v = mins[nd][0][j];
            else if (j < 2 * m) v = mins[nd][1][j - m];
            else v = mins[nd][2][j - 2 * m];
            S.cand[static_cast<size_t>(b0 + nd) * (3 * cap) + j] = v;
        }
        if (tid == 0) {
            for (int i = 0; i < NB; ++i)
                if (sm_m[i] > 0) {
                    ++my_joins;
                    my_m += static_cast<unsigned long long>(sm_m[i]);
                    my_q += static_cast<unsigned long long>(sm_q[i]);
                }
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

template <typename T, int MET, int NB>
constexpr size_t join_smem_bytes() {
    using E = typename std::conditional<MET == kMetCos, float, T>::type;
    return sizeof(E) * 2 * NB * kMaxSlots * SlabCfg<T>::kStride;
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
                if (key < G.kth_t[t]) {  // else it cannot enter G[t] (exact, D17)
                    atomicAdd(&c_app, 1u);
                    if (G.rec_cnt) {  // record mode (distributed refine)
                        const unsigned long long slot = atomicAdd(G.rec_cnt, 1ull);
                        G.rec_key[slot] = key;
                        G.rec_tgt[slot] = t;
                    } else {
                        const uint32_t slot = atomicAdd(G.bcnt + t, 1u);
                        G.bucket[G.boff[t] + slot] = key;
                    }
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
