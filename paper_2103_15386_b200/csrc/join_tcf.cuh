// join_tcf.cuh -- local join for float rows (L2 and cosine) with the distance
// tile on the 5th-generation tensor cores (Alg. 1 lines 9-31) and
// an EXACT selection: bit-identical to the canonical CUDA-core join.
//
// The batch layout, planning warp, gathers, TMEM row scans and fused filing
// are those of k_join_tc (join_tc.cuh); what changes is the arithmetic:
//
//   Gram = S S^T by tcgen05.mma.kind::tf32 (M = N = 128, K = 8 per
//   instruction; the fp32 rows staged in shared memory are read as TF32, i.e.
//   with their low 13 mantissa bits ignored), accumulator fp32 in TMEM.
//
//   For sample row s and column c:  v_c = n_c - 2 G_sc  (n = ||row||^2 in
//   fp32), so n_s + v_c approximates the squared distance D_sc (for unit
//   rows, twice the cosine distance).  A-priori bound: every operand carries a
//   relative error <= 2^-10 (truncation to TF32), so |G~ - G| <= (2^-9 + eps)
//   sum |a_i b_i| <= 2^-8.9 ||a|| ||b||, and |d~ - D| <= 2^-8.9 (n_s + n_c);
//   the canonical fp32 value differs from D by far less.  With
//   tau = 2^-7 (a 4x margin) every column whose canonical distance could be
//   the row minimum satisfies
//       v_c - tau n_c  <=  v_min + tau n_argmin + 2 tau n_s   (the window),
//   where v_min is the smallest v over the row's column set.
//
//   GetNearestObject (Alg. 2) per output: the window members' distances are
//   recomputed CANONICALLY (D5: acc = fmaf(x_i - y_i, x_i - y_i, acc) in
//   dimension order; D6 for cosine) from the fp32 rows in shared memory and
//   the smallest (dist, id) key wins -- the same key the CUDA-core tile
//   selects, so graphs stay bit-identical to the oracle.  Usually the window
//   holds the minimum alone.
//
// The rows of batch b must stay in shared memory for the recomputation, so
// the gather of batch b+2 is issued after the scans of b (join_tc.cuh issues
// it as soon as the MMA has read them).  KA = ceil(d / 32) K-atoms of 128-B
// rows (SW128 K-major, 16 KB per atom per batch); d % 4 == 0, d <= 128.
#pragma once
#include "join_tc.cuh"

namespace knng {

template <int KA>
struct TcfCfg {
    static constexpr size_t kAtom = static_cast<size_t>(kTcRows) * 128;     // 32 fp32 of 128 rows
    static constexpr size_t kRowBytes = KA * kAtom;                          // one batch
    static constexpr size_t kNrmOff = 2 * kRowBytes;                         // float n_c [3][128]
    static constexpr size_t kSideOff = kNrmOff + 3 * kTcRows * 4;            // u32 [3][4]
    static constexpr size_t kPlanOff = kSideOff + 3 * 4 * 4;
    static constexpr size_t kCacheOff = (kPlanOff + kTcPlans * sizeof(TcPlan) + 15) & ~size_t(15);
    static constexpr size_t kCacheCnt = 2 * 64;
    static constexpr size_t kCacheBytes = kCacheCnt + 2 * 32 * 2 * 32 * sizeof(uint32_t);
    static constexpr size_t kBarOff = (kCacheOff + kCacheBytes + 7) & ~size_t(7);
    static constexpr size_t kUsed = kBarOff + 8 * (1 + 2 * kTcPlans) + 8;
    static constexpr size_t kSmem = kUsed + 1024;
    static constexpr int kCtas = 2 * (kSmem + 1024) <= 233472 ? 2 : 1;
    static_assert(kSmem + 1024 <= 233472, "one CTA per SM at least");
};

// kind::tf32, tf32 x tf32 -> f32, K-major A and B, M = N = 128
constexpr uint32_t kTcfIdesc = (1u << 4) | (2u << 7) | (2u << 10) | ((128u >> 3) << 17) | ((128u >> 4) << 24);
constexpr float kTcfTau = 0.0078125f;  // 2^-7

__device__ __forceinline__ void tc_mma_tf32(uint32_t tmem, uint64_t ad, uint64_t bd, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
        "l"(ad), "l"(bd), "r"(kTcfIdesc), "r"(accumulate));
}

// canonical distance of staged rows a and b (slots), dims in order (D5 / D6)
template <int KA, bool COS>
__device__ __forceinline__ float tcf_canon(const unsigned char* rows, int a, int b, int d) {
    float acc = 0.0f;
    const int nch = d >> 2;  // 16-B chunks of 4 dims
#pragma unroll
    for (int at = 0; at < KA; ++at) {
        const unsigned char* ra = rows + at * TcfCfg<KA>::kAtom + a * 128;
        const unsigned char* rb = rows + at * TcfCfg<KA>::kAtom + b * 128;
#pragma unroll
        for (int ch = 0; ch < 8; ++ch) {
            if (at * 8 + ch >= nch) break;
            const float4 x = *reinterpret_cast<const float4*>(ra + ((ch ^ (a & 7)) << 4));
            const float4 y = *reinterpret_cast<const float4*>(rb + ((ch ^ (b & 7)) << 4));
            if constexpr (COS) {
                acc = fmaf(x.x, y.x, acc);
                acc = fmaf(x.y, y.y, acc);
                acc = fmaf(x.z, y.z, acc);
                acc = fmaf(x.w, y.w, acc);
            } else {
                float t;
                t = x.x - y.x; acc = fmaf(t, t, acc);
                t = x.y - y.y; acc = fmaf(t, t, acc);
                t = x.z - y.z; acc = fmaf(t, t, acc);
                t = x.w - y.w; acc = fmaf(t, t, acc);
            }
        }
    }
    if constexpr (COS) {
        const float r = 1.0f - acc;
        return r > 0.0f ? r : 0.0f;
    }
    return acc;
}

template <int KA, bool COS>
__global__ void __launch_bounds__(kTcThreads, TcfCfg<KA>::kCtas)
k_join_tcf(const float* __restrict__ X, const float* __restrict__ sqn, Dims D, Graph G, Samples S, int64_t boundary,
           unsigned long long* __restrict__ work, DevStats* __restrict__ stats) {
    using Cfg = TcfCfg<KA>;
    extern __shared__ __align__(16) unsigned char tc_raw[];
    unsigned char* tc_smem = tc_raw + ((1024 - (smem_u32(tc_raw) & 1023)) & 1023);
    unsigned char* rows = tc_smem;
    float* nrm = reinterpret_cast<float*>(tc_smem + Cfg::kNrmOff);
    uint32_t* side = reinterpret_cast<uint32_t*>(tc_smem + Cfg::kSideOff);
    TcPlan* plans = reinterpret_cast<TcPlan*>(tc_smem + Cfg::kPlanOff);
    uint8_t* cc_cnt = tc_smem + Cfg::kCacheOff;
    uint32_t* cc_ids = reinterpret_cast<uint32_t*>(tc_smem + Cfg::kCacheOff + Cfg::kCacheCnt);
    uint64_t* mma_bar = reinterpret_cast<uint64_t*>(tc_smem + Cfg::kBarOff);
    uint64_t* plan_full = mma_bar + 1;
    uint64_t* plan_empty = plan_full + kTcPlans;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(plan_empty + kTcPlans);

    const int tid = threadIdx.x;
    const int warp = tid >> 5;
    const uint32_t lane = lane_id();
    const int d = D.d, cap = D.cap;
    const bool restricted = boundary >= 0;

    // ---------------------------------------------------------------- plans
    int cbuf = 1;
    uint32_t pend = 0;
    int64_t xnext = 0;
    unsigned long long claimed = 0;
    int my_m = 0, my_q = 0;
    bool more = true;
    unsigned long long n_joins = 0, n_m = 0, n_q = 0;
    auto claim = [&]() -> unsigned long long {
        unsigned long long c0 = 0;
        if (lane == 0) c0 = atomicAdd(work, 32ull);
        return c0;
    };
    auto fetch = [&](int buf, int64_t xb) {
        if (xb < D.n) {
            const int nodes = static_cast<int>(D.n - xb < 32 ? D.n - xb : 32);
            if (lane < 16) {
                const int lo = 4 * static_cast<int>(lane), bytes = max(0, min(4, 2 * nodes - lo));
                asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(smem_u32(cc_cnt + buf * 64 + lo)),
                             "l"(S.gcnt + 2 * xb + lo), "r"(bytes)
                             : "memory");
            }
            uint32_t* cids = cc_ids + static_cast<size_t>(buf) * 32 * 2 * cap;
            if ((cap & 3) == 0) {
                if (static_cast<int>(lane) < nodes) {
                    const uint32_t* gn = S.G + static_cast<size_t>(xb + lane) * cap;
                    const uint32_t* go = gn + static_cast<size_t>(D.n) * cap;
                    const uint32_t dn = smem_u32(cids + lane * 2 * cap), dq = dn + 4 * cap;
                    for (int c = 0; c < cap; c += 4) {
                        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dn + 4 * c), "l"(gn + c)
                                     : "memory");
                        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dq + 4 * c), "l"(go + c)
                                     : "memory");
                    }
                }
            } else {
                for (int e = lane; e < nodes * 2 * cap; e += 32) {
                    const int node = e / (2 * cap), w = e - node * 2 * cap;
                    const uint32_t* src = w < cap ? S.G + static_cast<size_t>(xb + node) * cap + w
                                                  : S.G + static_cast<size_t>(D.n) * cap +
                                                        static_cast<size_t>(xb + node) * cap + (w - cap);
                    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(smem_u32(cids + e)), "l"(src)
                                 : "memory");
                }
            }
        }
        cp_async_commit();
    };
    auto advance = [&]() -> bool {
        if (xnext >= D.n) return false;
        cp_async_wait<0>();
        __syncwarp();
        cbuf ^= 1;
        my_m = 0;
        my_q = 0;
        if (xnext + lane < D.n) {
            my_m = cc_cnt[cbuf * 64 + 2 * lane];
            my_q = cc_cnt[cbuf * 64 + 2 * lane + 1];
        }
        if (my_m == 0) my_q = 0;
        pend = __ballot_sync(kFull, my_m > 0);
        xnext = static_cast<int64_t>(__shfl_sync(kFull, claimed, 0));
        claimed = claim();
        fetch(cbuf ^ 1, xnext);
        return true;
    };
    auto form_plan = [&](TcPlan& P) {
        while (pend == 0) {
            if (!more || !advance()) {
                more = false;
                if (lane == 0) P.nnodes = 0;
                __syncwarp();  // the terminator is read by every lane
                return;
            }
        }
        const uint32_t* cids = cc_ids + static_cast<size_t>(cbuf) * 32 * 2 * cap;
        int ns_used = 0, nn = 0;
        while (true) {
            const bool fit = ((pend >> lane) & 1u) && my_m + my_q <= kTcRows - ns_used;
            const uint32_t fm = __ballot_sync(kFull, fit);
            if (fm == 0) break;
            const int L = __ffs(fm) - 1;
            const int m = __shfl_sync(kFull, my_m, L), q = __shfl_sync(kFull, my_q, L);
            if (static_cast<int>(lane) == L) {
                P.sb[nn] = ns_used;
                P.m[nn] = m;
                P.q[nn] = q;
                ++n_joins;
                n_m += m;
                n_q += q;
            }
            const uint32_t* row = cids + L * 2 * cap;
            for (int js = lane; js < m + q; js += 32) {
                P.ids[ns_used + js] = js < m ? row[js] : row[cap + (js - m)];
                P.map[ns_used + js] = static_cast<uint8_t>(nn);
            }
            ns_used += m + q;
            pend &= ~(1u << L);
            ++nn;
        }
        for (int js = ns_used + lane; js < kTcRows; js += 32) {
            P.ids[js] = 0xFFFFFFFFu;
            P.map[js] = 0xFF;
        }
        if (lane == 0) {
            P.nnodes = nn;
            P.nslots = ns_used;
        }
        __syncwarp();
    };

    // ------------------------------------------------------------- gathers
    // thread t (< 128) copies 16-B chunk (t & 7) of every K-atom of slots
    // (t >> 3) + 16 i into the SW128 layout; chunks past d/4 are zero-filled
    const int part = tid & 7, row0 = tid >> 3;
    const int nchunks = d >> 2;
    float nv_next = 0.0f;
    uint32_t side_next = 0;
    auto gather = [&](const TcPlan& P, unsigned char* dst) {
        const int nslots = P.nslots;
        const uint32_t dbase = smem_u32(dst);
#pragma unroll
        for (int at = 0; at < KA; ++at) {
            const int c = at * 8 + part;
            const uint32_t abase = dbase + at * static_cast<uint32_t>(Cfg::kAtom);
            if (c < nchunks) {
                const float* src0 = X + c * 4;
                for (int slot = row0; slot < nslots; slot += 16) {
                    const uint32_t id = P.ids[slot];
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(
                                     abase + slot * 128 + ((part ^ (slot & 7)) << 4)),
                                 "l"(src0 + static_cast<size_t>(id) * d)
                                 : "memory");
                }
            } else {
                for (int slot = row0; slot < nslots; slot += 16)
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, 0;\n" ::"r"(
                                     abase + slot * 128 + ((part ^ (slot & 7)) << 4)),
                                 "l"(X)
                                 : "memory");
            }
        }
        cp_async_commit();
        const uint32_t id = P.ids[tid];
        nv_next = id != 0xFFFFFFFFu ? __ldg(sqn + id) : 0.0f;
        side_next = __ballot_sync(kFull, id != 0xFFFFFFFFu && static_cast<int64_t>(id) >= boundary);
    };

    // --------------------------------------------------------------- filing
    uint64_t f1_key[2], f1_th = 0, f1_bo = 0;
    uint32_t f1_tgt = 0;
    uint64_t f2_key[2], f2_pos[2];
    uint32_t f2_tgt = 0;
#pragma unroll
    for (int r = 0; r < 2; ++r) {
        f1_key[r] = kSentinel;
        f2_key[r] = kSentinel;
        f2_pos[r] = 0;
    }
    unsigned long long n_cand = 0, n_app = 0, my_pairs = 0, n_recomp = 0;
    auto file_store = [&]() {
#pragma unroll
        for (int r = 0; r < 2; ++r)
            if (f2_key[r] != kSentinel) {
                if (G.rec_cnt) {  // record mode (distributed refine)
                    G.rec_key[f2_pos[r]] = f2_key[r];
                    G.rec_tgt[f2_pos[r]] = f2_tgt;
                } else {
                    G.bucket[f2_pos[r]] = f2_key[r];
                }
            }
    };
    auto file_atomic = [&]() {
        const bool ok0 = f1_key[0] < f1_th, ok1 = f1_key[1] < f1_th;  // D17
        n_app += ok0 + ok1;
        uint64_t sl = 0;
        if (G.rec_cnt) {
            // record slots: one atomic per warp (the call is warp-uniform)
            const uint32_t b0 = __ballot_sync(kFull, ok0), b1 = __ballot_sync(kFull, ok1);
            unsigned long long wb = 0;
            if (lane == 0 && (b0 | b1)) wb = atomicAdd(G.rec_cnt, static_cast<unsigned long long>(__popc(b0) + __popc(b1)));
            sl = shfl_u64(wb, 0) + __popc(b0 & lanemask_lt()) + __popc(b1 & lanemask_lt());
            f1_bo = 0;
            f2_tgt = f1_tgt;
        } else if (ok0 || ok1) {
            sl = atomicAdd(G.bcnt + f1_tgt, static_cast<uint32_t>(ok0 + ok1));
        }
        f2_key[0] = ok0 ? f1_key[0] : kSentinel;
        f2_pos[0] = f1_bo + sl;
        f2_key[1] = ok1 ? f1_key[1] : kSentinel;
        f2_pos[1] = f1_bo + sl + (ok0 ? 1 : 0);
        f1_key[0] = kSentinel;
        f1_key[1] = kSentinel;
        f1_th = 0;
    };

    // ------------------------------------------------------------- prologue
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(kTcRows)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (tid == 0) {
        mbar_init(mma_bar, 1);
        for (int i = 0; i < kTcPlans; ++i) {
            mbar_init(plan_full + i, 1);
            mbar_init(plan_empty + i, kTcPlanWarp);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == kTcPlanWarp) {
        xnext = static_cast<int64_t>(__shfl_sync(kFull, claim(), 0));
        claimed = claim();
        fetch(0, xnext);
        for (uint32_t t = 0;; ++t) {
            const int slot = t % kTcPlans;
            if (t >= kTcPlans) mbar_wait_suspend(plan_empty + slot, ((t / kTcPlans) - 1) & 1);
            form_plan(plans[slot]);
            const bool last = plans[slot].nnodes == 0;
            if (lane == 0) mbar_arrive(plan_full + slot);
            if (last) break;
        }
    } else {
        bool ended = false;
        for (int t = 0; t < 2; ++t) {
            if (!ended) {
                mbar_wait(plan_full + t, 0);
                ended = plans[t].nnodes == 0;
            }
            if (!ended) gather(plans[t], rows + t * Cfg::kRowBytes);
            else cp_async_commit();
            if (t == 0) {
                nrm[tid] = nv_next;
                if (lane == 0) side[warp] = side_next;
            }
        }
        for (uint32_t b = 0;; ++b) {
            const int slot = b % kTcPlans;
            const TcPlan& P = plans[slot];
            const int buf = b & 1;
            const unsigned char* myrows = rows + buf * Cfg::kRowBytes;
            if (P.nnodes == 0) break;
            cp_async_wait<1>();
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            named_bar(1, kTcPlanWarp * 32);  // rows(b) visible; TMEM reads and row reads of b-1 done
            if (tid == 0) {
                tc_fence_after();
                const uint32_t base = smem_u32(myrows);
#pragma unroll
                for (int k = 0; k < 4 * KA; ++k) {
                    const uint64_t desc = tc_smem_desc(base + (k >> 2) * static_cast<uint32_t>(Cfg::kAtom) + 32 * (k & 3));
                    tc_mma_tf32(tmem, desc, desc, k > 0 ? 1u : 0u);
                }
                tc_commit(mma_bar);
            }

            const int s = tid;
            const int nd = P.map[s];
            bool isNEW = false, isOLD = false;
            int sb = 0, m = 0, q = 0;
            if (nd != 0xFF) {
                sb = P.sb[nd];
                m = P.m[nd];
                q = P.q[nd];
                isNEW = s - sb < m;
                isOLD = !isNEW;
            }
            const bool act = isNEW || isOLD;
            const int lo = act ? sb : kTcRows;
            const int hi = act ? (isNEW ? sb + m + q : sb + m) : 0;
            const int wlo = __reduce_min_sync(kFull, lo), whi = __reduce_max_sync(kFull, hi);
            const uint32_t my_id = P.ids[s];
            const bool myside = restricted && static_cast<int64_t>(my_id) >= boundary;
            const int nbuf = b % 3;
            const float* nb = nrm + nbuf * kTcRows;
            const float ns = nb[s];
            mbar_wait(mma_bar, b & 1);
            tc_fence_after();

            // column masks of one 16-column chunk (A: NEW-or-NEW-other set, B: OLD set)
            auto masks = [&](int cb, uint32_t& A, uint32_t& B) {
                A = act ? bit_range(sb - cb, sb + m - cb) : 0u;
                if (isNEW && s >= cb && s < cb + 16) A &= ~(1u << (s - cb));
                B = isNEW ? bit_range(sb + m - cb, sb + m + q - cb) : 0u;
                if (restricted) {
                    const uint32_t sd = side[nbuf * 4 + (cb >> 5)] >> (cb & 16);
                    const uint32_t allow = myside ? ~sd : sd;
                    A &= allow;
                    B &= allow;
                }
                A &= 0xFFFFu;
                B &= 0xFFFFu;
            };
            // pass 1: approximate minima v = n_c - 2 G and their columns
            float vA = INFINITY, vB = INFINITY;
            int cA = -1, cB = -1;
            for (int cb = wlo & ~15; cb < whi; cb += 16) {
                uint32_t r[16];
                tc_ld16(tmem + (static_cast<uint32_t>(warp * 32) << 16) + cb, r);
                uint32_t A, B;
                masks(cb, A, B);
                if (isNEW) my_pairs += __popc(A & bit_range(0, s - cb)) + __popc(B);
#pragma unroll
                for (int e = 0; e < 16; ++e) {
                    const float v = fmaf(-2.0f, __uint_as_float(r[e]), nb[cb + e]);
                    if (((A >> e) & 1u) && v < vA) { vA = v; cA = cb + e; }
                    if (((B >> e) & 1u) && v < vB) { vB = v; cB = cb + e; }
                }
            }
            // window thresholds (see the header); cosine rows have n ~ 1
            const float slack = COS ? 0x1p-16f : 0.0f;
            const float tA = cA >= 0 ? vA + kTcfTau * (nb[cA] + 2.0f * ns) + slack : -INFINITY;
            const float tB = cB >= 0 ? vB + kTcfTau * (nb[cB] + 2.0f * ns) + slack : -INFINITY;
            // pass 2: canonical recomputation of the window members
            uint64_t k1 = kSentinel, k2 = kSentinel;
            for (int cb = wlo & ~15; cb < whi; cb += 16) {
                uint32_t r[16];
                tc_ld16(tmem + (static_cast<uint32_t>(warp * 32) << 16) + cb, r);
                uint32_t A, B;
                masks(cb, A, B);
                uint32_t W = 0;
#pragma unroll
                for (int e = 0; e < 16; ++e) {
                    const float lowr = fmaf(-2.0f, __uint_as_float(r[e]), nb[cb + e]) - kTcfTau * nb[cb + e];
                    if (((A >> e) & 1u) && lowr <= tA) W |= 1u << e;
                    if (((B >> e) & 1u) && lowr <= tB) W |= 1u << (16 + e);
                }
                while (W) {
                    const int bit = __ffs(W) - 1;
                    W &= W - 1;
                    const int col = cb + (bit & 15);
                    const uint64_t kk = make_key(tcf_canon<KA, COS>(myrows, s, col, d), P.ids[col]);
                    ++n_recomp;
                    if (bit < 16) k1 = kk < k1 ? kk : k1;
                    else k2 = kk < k2 ? kk : k2;
                }
            }
            tc_fence_before();

            // ---- deferred filing of the two previous batches, then this one's keys
            file_store();
            file_atomic();
            f1_key[0] = act ? k1 : kSentinel;
            f1_key[1] = isNEW ? k2 : kSentinel;
            f1_tgt = my_id;
            n_cand += (f1_key[0] != kSentinel) + (f1_key[1] != kSentinel);
            if (f1_key[0] != kSentinel || f1_key[1] != kSentinel) {  // D15
                f1_th = __ldg(G.kth_t + my_id);
                if (!G.rec_cnt) f1_bo = __ldg(G.boff + my_id);
            }
            // rows(b) are no longer read by this warp: after every warp is
            // here (named barrier at the top of b+1 orders it), gather b+2
            // into them.  Norms of b+1 (loaded one iteration ago) are staged.
            // (nv_next / side_next still hold batch b+1's, gathered at b-1)
            __syncwarp();
            nrm[((b + 1) % 3) * kTcRows + tid] = nv_next;
            if (lane == 0) side[((b + 1) % 3) * 4 + warp] = side_next;
            named_bar(2, kTcPlanWarp * 32);  // all row reads of batch b done
            if (!ended) {
                const int s2 = (b + 2) % kTcPlans;
                mbar_wait(plan_full + s2, ((b + 2) / kTcPlans) & 1);
                ended = plans[s2].nnodes == 0;
            }
            if (!ended) gather(plans[(b + 2) % kTcPlans], rows + buf * Cfg::kRowBytes);
            else cp_async_commit();
            if (lane == 0) mbar_arrive(plan_empty + slot);  // this warp is done with plan b
        }
    }
    if (warp < kTcPlanWarp) {
        file_store();
        file_atomic();
        file_store();
    }
    cp_async_wait<0>();
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTcRows) : "memory");
    }

#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        n_cand += __shfl_xor_sync(kFull, n_cand, o);
        n_app += __shfl_xor_sync(kFull, n_app, o);
        my_pairs += __shfl_xor_sync(kFull, my_pairs, o);
        n_joins += __shfl_xor_sync(kFull, n_joins, o);
        n_m += __shfl_xor_sync(kFull, n_m, o);
        n_q += __shfl_xor_sync(kFull, n_q, o);
        n_recomp += __shfl_xor_sync(kFull, n_recomp, o);
    }
    if (lane == 0) {
        if (n_cand) atomicAdd(&stats->candidates, n_cand);
        if (n_app) atomicAdd(&stats->appended, n_app);
        if (my_pairs) atomicAdd(&stats->dist_evals, my_pairs);
        if (n_recomp) atomicAdd(&stats->recomputed, n_recomp);
        if (warp == kTcPlanWarp && n_joins) {
            atomicAdd(&stats->joins, n_joins);
            atomicAdd(&stats->sum_m, n_m);
            atomicAdd(&stats->sum_q, n_q);
            atomicAdd(&stats->rows, n_m + n_q);
        }
    }
}

// fp32 squared norms (any order: they only feed the approximate tile)
__global__ void k_sqnorm_f32(const float* __restrict__ X, int64_t n, int d, float* __restrict__ out) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float* x = X + i * d;
    float acc = 0.0f;
    for (int j = 0; j < d; ++j) acc = fmaf(x[j], x[j], acc);
    out[i] = acc;
}

}  // namespace knng
