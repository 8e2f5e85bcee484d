// join_ws.cuh -- warp-specialised local join (Alg. 1 lines 9-31).
//
// Same computation as k_join (join_kernel.cuh), organised as a producer /
// consumer pipeline for sm_100a:
//
//  producer warp : grabs chunks of 32 nodes from a global work counter,
//                  packs consecutive nodes into a batch whose 4x4 register
//                  blocks fit the 256 consumer threads (one block each) and
//                  whose sample rows fit one ring stage, publishes the batch
//                  metadata (ids, node offsets) into a 2-entry metadata ring,
//                  then for every 32-dim slab issues one cp.async.bulk copy
//                  per sample row (UBLKCP: global -> shared, completion via
//                  an mbarrier transaction count) into a STAGES-deep ring.
//  consumer warps: 8 warps; each thread owns one 4x4 block of the batch's
//                  tiles (NEW rows x sample columns), accumulates the
//                  canonical distance (D5/D6) slab by slab as the ring fills,
//                  releases each stage with one mbarrier arrive per warp,
//                  then runs GetNearestObject (packed-key shared atomicMin,
//                  P:237) and writes the 2m+q selected keys per node.
//
// No CTA-wide barrier sits on the slab path: gathers of batch b+1 overlap
// the tiles of batch b, and the per-chunk address arithmetic of the
// cp.async version is replaced by one bulk-copy instruction per row slab.
#pragma once
#include "join_kernel.cuh"

namespace knng {

constexpr int kWsConsumerWarps = 8;
constexpr int kWsThreads = (kWsConsumerWarps + 1) * 32;
constexpr int kWsSlots = 256;    // sample rows per stage (all nodes of a batch)
constexpr int kWsBlocks = kWsConsumerWarps * 32;  // 4x4 blocks per batch
constexpr int kWsMaxNodes = 32;  // nodes per batch (one producer chunk)
constexpr int kWsMeta = 2;

struct WsMeta {
    int nnodes;   // 0 = no more work
    int nblocks;
    int nslots;
    int pad_;
    int64_t x[kWsMaxNodes];
    int m[kWsMaxNodes], q[kWsMaxNodes], sbase[kWsMaxNodes], bbase[kWsMaxNodes + 1];
    uint32_t ids[kWsSlots];
    unsigned long long mnA[kWsSlots];  // c_nn of a NEW slot, c_on of an OLD slot
    unsigned long long mnB[kWsSlots];  // c_no of a NEW slot
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t tx) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(smem_u32(bar)),
                 "r"(tx)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

template <typename T, bool COS, int STAGES>
struct WsCfg {
    using E = typename std::conditional<COS, float, T>::type;
    static constexpr int SD = SlabCfg<T>::kDims;
    static constexpr int RS = SlabCfg<T>::kStride;
    static constexpr size_t kStageBytes = sizeof(E) * kWsSlots * RS;
    static constexpr size_t kMetaOff = kStageBytes * STAGES;
    static constexpr size_t kBarOff = (kMetaOff + sizeof(WsMeta) * kWsMeta + 15) & ~size_t(15);
    static constexpr size_t kSmem = kBarOff + 8 * (2 * STAGES + 2 * kWsMeta);
};

template <typename T, bool COS, int STAGES>
__global__ void __launch_bounds__(kWsThreads, 1)
k_join_ws(const T* __restrict__ X, const float* __restrict__ Xn, Dims D, Samples S, int64_t boundary,
          unsigned long long* __restrict__ work, DevStats* __restrict__ stats) {
    using Cfg = WsCfg<T, COS, STAGES>;
    using E = typename Cfg::E;
    constexpr bool kFloat = std::is_same<E, float>::value;
    using Acc = typename std::conditional<kFloat, float, unsigned int>::type;
    constexpr int SD = Cfg::SD, RS = Cfg::RS;
    const E* __restrict__ V = COS ? reinterpret_cast<const E*>(Xn) : reinterpret_cast<const E*>(X);

    extern __shared__ __align__(128) unsigned char ws_smem[];
    E* ring = reinterpret_cast<E*>(ws_smem);
    WsMeta* meta = reinterpret_cast<WsMeta*>(ws_smem + Cfg::kMetaOff);
    uint64_t* bars = reinterpret_cast<uint64_t*>(ws_smem + Cfg::kBarOff);
    uint64_t* full = bars;                    // [STAGES]
    uint64_t* empty = bars + STAGES;          // [STAGES]
    uint64_t* mfull = bars + 2 * STAGES;      // [kWsMeta]
    uint64_t* mempty = bars + 2 * STAGES + kWsMeta;

    const int tid = threadIdx.x;
    const int warp = tid >> 5;
    const uint32_t lane = lane_id();
    const int d = D.d, cap = D.cap;
    const int nslab = (d + SD - 1) / SD;

    if (tid == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, kWsConsumerWarps);
        }
        for (int s = 0; s < kWsMeta; ++s) {
            mbar_init(mfull + s, 32);
            mbar_init(mempty + s, 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (warp == kWsConsumerWarps) {
        // =============================== producer ===============================
        uint32_t slab_it = 0, meta_it = 0;
        int64_t x0 = 0;
        int cur = 32;  // position inside the current 32-node chunk
        int my_m = 0, my_q = 0, my_nb = 0, my_sl = 0;
        unsigned long long n_joins = 0, n_m = 0, n_q = 0;
        while (true) {
            if (cur >= 32) {
                unsigned long long c0 = 0;
                if (lane == 0) c0 = atomicAdd(work, 32ull);
                x0 = static_cast<int64_t>(__shfl_sync(kFull, c0, 0));
                if (x0 >= D.n) break;
                const int64_t x = x0 + lane;
                my_m = 0;
                my_q = 0;
                if (x < D.n) {
                    my_m = S.gcnt[2 * x];
                    my_q = S.gcnt[2 * x + 1];
                }
                if (my_m == 0) my_q = 0;  // no NEW sample: nothing to join
                const int mg = (my_m + 3) >> 2, qg = (my_q + 3) >> 2;
                my_nb = mg * (mg + 1) / 2 + mg * qg;
                my_sl = 4 * (mg + qg);
                cur = 0;
            }
            // take nodes cur.. while the batch's blocks and slots fit
            const bool pending = static_cast<int>(lane) >= cur;
            int cb = pending ? my_nb : 0, cs = pending ? my_sl : 0;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int tb = __shfl_up_sync(kFull, cb, o), ts = __shfl_up_sync(kFull, cs, o);
                if (static_cast<int>(lane) >= o) { cb += tb; cs += ts; }
            }
            const bool fits = pending && cb <= kWsBlocks && cs <= kWsSlots;
            const uint32_t fm = __ballot_sync(kFull, fits);
            const int end = fm ? 32 - __clz(fm) : cur;  // fits is a prefix of [cur, 32)
            const int nb_tot = __shfl_sync(kFull, cb, end - 1 < 0 ? 0 : end - 1);
            const int ns_tot = __shfl_sync(kFull, cs, end - 1 < 0 ? 0 : end - 1);
            const int first = cur;
            cur = end;
            if (nb_tot == 0) continue;  // only nodes without NEW samples
            // ---- publish batch metadata
            const int mb = meta_it % kWsMeta;
            mbar_wait(mempty + mb, ((meta_it / kWsMeta) & 1) ^ 1);
            WsMeta& M = meta[mb];
            const int nn = end - first;
            const int excl_b = cb - (pending ? my_nb : 0), excl_s = cs - (pending ? my_sl : 0);
            if (static_cast<int>(lane) >= first && static_cast<int>(lane) < end) {
                const int i = lane - first;
                M.x[i] = x0 + lane;
                M.m[i] = my_m;
                M.q[i] = my_q;
                M.sbase[i] = excl_s;
                M.bbase[i] = excl_b;
                if (my_m > 0) {
                    ++n_joins;
                    n_m += my_m;
                    n_q += my_q;
                }
            }
            if (lane == 0) {
                M.nnodes = nn;
                M.nblocks = nb_tot;
                M.nslots = ns_tot;
                M.bbase[nn] = nb_tot;
            }
            int rows = 0;
            for (int i = 0; i < nn; ++i) {
                const int src = first + i;
                const int m = __shfl_sync(kFull, my_m, src), q = __shfl_sync(kFull, my_q, src);
                const int sb = __shfl_sync(kFull, excl_s, src);
                const int mpad = (m + 3) & ~3, qpad = (q + 3) & ~3;
                const int64_t x = x0 + src;
                for (int j = lane; j < mpad + qpad; j += 32) {
                    uint32_t id = 0xFFFFFFFFu;
                    if (j < m) id = S.G[static_cast<size_t>(x) * cap + j];
                    else if (j >= mpad && j - mpad < q)
                        id = S.G[static_cast<size_t>(D.n) * cap + static_cast<size_t>(x) * cap + (j - mpad)];
                    M.ids[sb + j] = id;
                    M.mnA[sb + j] = kSentinel;
                    M.mnB[sb + j] = kSentinel;
                }
                rows += m + q;
            }
            __syncwarp();
            mbar_arrive(mfull + mb);  // all 32 lanes: releases every lane's writes
            ++meta_it;
            // ---- gathers: one bulk copy per valid row per slab
            for (int sl = 0; sl < nslab; ++sl) {
                const int st = slab_it % STAGES;
                mbar_wait(empty + st, ((slab_it / STAGES) & 1) ^ 1);
                const int d0 = sl * SD;
                const uint32_t rb = static_cast<uint32_t>(min(SD, d - d0) * sizeof(E));
                if (lane == 0) mbar_arrive_expect_tx(full + st, rb * static_cast<uint32_t>(rows));
                __syncwarp();
                E* dst = ring + static_cast<size_t>(st) * kWsSlots * RS;
                for (int j = lane; j < ns_tot; j += 32) {
                    const uint32_t id = M.ids[j];
                    if (id != 0xFFFFFFFFu) bulk_g2s(dst + j * RS, V + static_cast<size_t>(id) * d + d0, rb, full + st);
                }
                ++slab_it;
            }
        }
        // termination marker
        const int mb = meta_it % kWsMeta;
        mbar_wait(mempty + mb, ((meta_it / kWsMeta) & 1) ^ 1);
        if (lane == 0) meta[mb].nnodes = 0;
        __syncwarp();
        mbar_arrive(mfull + mb);
        // stats
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            n_joins += __shfl_xor_sync(kFull, n_joins, o);
            n_m += __shfl_xor_sync(kFull, n_m, o);
            n_q += __shfl_xor_sync(kFull, n_q, o);
        }
        if (lane == 0 && n_joins) {
            atomicAdd(&stats->joins, n_joins);
            atomicAdd(&stats->sum_m, n_m);
            atomicAdd(&stats->sum_q, n_q);
            atomicAdd(&stats->rows, n_m + n_q);
        }
        return;
    }

    // ================================ consumers =================================
    const int ct = tid;  // 0 .. kWsBlocks-1
    uint32_t slab_it = 0, meta_it = 0;
    unsigned long long my_pairs = 0;
    while (true) {
        const int mb = meta_it % kWsMeta;
        mbar_wait(mfull + mb, (meta_it / kWsMeta) & 1);
        const WsMeta& M = meta[mb];
        const int nn = M.nnodes;
        if (nn == 0) break;
        // ---- my block
        const bool active = ct < M.nblocks;
        int nd = 0;
        if (active)
            while (nd + 1 < nn && M.bbase[nd + 1] <= ct) ++nd;
        const int m = M.m[nd], q = M.q[nd], sb = M.sbase[nd];
        const int mpad = (m + 3) & ~3, mg = mpad >> 2, qg = (q + 3) >> 2;
        const int t = ct - M.bbase[nd];
        const int nnn = mg * (mg + 1) / 2;
        int I = 0, J = 0;
        if (active) {
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
        const bool nn_blk = J < mg;
        const int rb = 4 * I;
        const int cb = nn_blk ? 4 * J : mpad + 4 * (J - mg);
        const int aoff = (sb + rb) * RS, boff = (sb + cb) * RS;

        Acc acc[4][4];
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
            for (int c = 0; c < 4; ++c) acc[r][c] = Acc(0);

        for (int sl = 0; sl < nslab; ++sl) {
            const int st = slab_it % STAGES;
            mbar_wait(full + st, (slab_it / STAGES) & 1);
            if (active) {
                const E* __restrict__ A = ring + static_cast<size_t>(st) * kWsSlots * RS + aoff;
                const E* __restrict__ B = ring + static_cast<size_t>(st) * kWsSlots * RS + boff;
                const int lim = min(SD, d - sl * SD);
                if constexpr (kFloat) {
#pragma unroll
                    for (int i = 0; i < SD; i += 4) {
                        if (i >= lim) break;
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
                                    float tt;
                                    tt = a[r].x - b[c].x; acc[r][c] = fmaf(tt, tt, acc[r][c]);
                                    tt = a[r].y - b[c].y; acc[r][c] = fmaf(tt, tt, acc[r][c]);
                                    tt = a[r].z - b[c].z; acc[r][c] = fmaf(tt, tt, acc[r][c]);
                                    tt = a[r].w - b[c].w; acc[r][c] = fmaf(tt, tt, acc[r][c]);
                                }
                            }
                    }
                } else {
#pragma unroll
                    for (int i = 0; i < SD; i += 4) {
                        if (i >= lim) break;
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
                                acc[r][c] = __dp4a(ad, ad, acc[r][c]);
                            }
                    }
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(empty + st);
            ++slab_it;
        }

        // ---- GetNearestObject (Alg. 2): pre-reduce, then shared atomicMin
        if (active) {
            const uint32_t* nid = M.ids + sb;
            unsigned long long* mnA = const_cast<unsigned long long*>(M.mnA) + sb;
            unsigned long long* mnB = const_cast<unsigned long long*>(M.mnB) + sb;
            uint64_t colbest[4] = {kSentinel, kSentinel, kSentinel, kSentinel};
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const int u = rb + r;
                uint64_t rowbest = kSentinel;
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const int w = cb + c;
                    bool valid = nn_blk ? (u < m && w < u) : (u < m && (w - mpad) < q);
                    if (valid) valid = allowed_pair(boundary, nid[u], nid[w]);
                    if (!valid) continue;
                    float dist;
                    if constexpr (COS) {
                        const float x1 = 1.0f - acc[r][c];
                        dist = x1 > 0.0f ? x1 : 0.0f;
                    } else if constexpr (kFloat) {
                        dist = acc[r][c];
                    } else {
                        dist = static_cast<float>(acc[r][c]);
                    }
                    ++my_pairs;
                    const uint64_t kr = make_key(dist, nid[w]);
                    const uint64_t kc = make_key(dist, nid[u]);
                    rowbest = kr < rowbest ? kr : rowbest;
                    colbest[c] = kc < colbest[c] ? kc : colbest[c];
                }
                if (rowbest != kSentinel) atomicMin(nn_blk ? &mnA[u] : &mnB[u], static_cast<unsigned long long>(rowbest));
            }
#pragma unroll
            for (int c = 0; c < 4; ++c)
                if (colbest[c] != kSentinel) atomicMin(&mnA[cb + c], static_cast<unsigned long long>(colbest[c]));
        }
        asm volatile("bar.sync 1, %0;" ::"n"(kWsBlocks) : "memory");
        // ---- output: slot j of node x: c_nn(u_j), c_no(u_j), c_on(w_j)
        for (int idx = ct; idx < nn * 96; idx += kWsBlocks) {
            const int i = idx / 96, j = idx - i * 96;
            const int mi = M.m[i], qi = M.q[i];
            if (j >= 2 * mi + qi) continue;
            const int sbi = M.sbase[i], mpi = (mi + 3) & ~3;
            uint64_t v;
            if (j < mi) v = M.mnA[sbi + j];
            else if (j < 2 * mi) v = M.mnB[sbi + j - mi];
            else v = M.mnA[sbi + mpi + (j - 2 * mi)];
            S.cand[static_cast<size_t>(M.x[i]) * (3 * cap) + j] = v;
        }
        asm volatile("bar.sync 1, %0;" ::"n"(kWsBlocks) : "memory");
        if (ct == 0) mbar_arrive(mempty + mb);
        ++meta_it;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) my_pairs += __shfl_xor_sync(kFull, my_pairs, o);
    if (lane == 0 && my_pairs) atomicAdd(&stats->dist_evals, my_pairs);
}

}  // namespace knng
