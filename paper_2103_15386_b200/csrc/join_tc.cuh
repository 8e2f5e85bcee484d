// join_tc.cuh -- local join on the 5th-generation tensor cores for uint8 rows
// of <= 128 dims (Alg. 1 lines 9-31; the exact-u8 path of D35).
//
// For integer vectors the canonical distance (D5) is an exact integer, and so
// is  ||a||^2 + ||b||^2 - 2 a.b  evaluated in int32: the two are the same
// number, so a Gram-matrix formulation is bit-identical to the oracle's
// sum of squared differences (d <= 128 keeps every value < 2^23).  The
// pairwise tile of a node's samples is therefore computed as
//
//     Gram = S S^T   (S: the batch's 128 staged sample rows, u8, K = d)
//
// by tcgen05.mma.kind::i8 (M = N = 128, K = 32 per instruction, accumulator
// in TMEM) instead of on the ALUs.  The batch packs whole nodes (first fit)
// into the 128 rows; only the diagonal blocks of the Gram matrix are used.
//
// Thread s of the 4 epilogue warps owns TMEM lane s = sample slot s and scans
// its own node's columns (tcgen05.ld, 16 columns at a time):
//   NEW sample u: c_nn(u) = min over the other NEW samples, c_no(u) = min
//                 over the OLD samples;
//   OLD sample w: c_on(w) = min over the NEW samples
// -- the GetNearestObject of Alg. 2 for every sample, as row minima of the
// full symmetric tile (the triangular tile + column minima of join_ws.cuh
// and join_ls.cuh give the same keys).  The key of column c is the int32
//     (n_c - 2 a.b) * 128 + c,
// whose order is the (dist, id) order of D3: dist = n_s + (n_c - 2 a.b) with
// n_s fixed per row, and inside the NEW (or OLD) segment of a node the slot
// order is the id order (k_rev_select writes both sample lists sorted, D11).
// With n'_c = n_c * 128 + c staged per batch, one IMAD per column forms it.
//
// CTA = EPI epilogue warps (4, or 8 in the default instance: 3 CTAs per SM)
// + 1 planning warp, 128 TMEM columns per CTA.  The planning warp fills a
// 4-deep plan ring (mbarrier hand-off) from the chunk cache, running ahead of
// the rest, and (TMA build, TC_PGATHER) issues each batch's row gathers once
// the MMA two batches back has released the row buffer.  Iteration b of the
// epilogue warps (two row buffers, two batches of rows in flight):
//     named barrier (TMEM reads of b-1 done, norms of b visible)
//     thread 0: wait rows(b); kch MMAs (K = 32 each) of batch b -> TMEM,
//       commit -> mbarrier(s)
//     filing of b-1 / b-2 while MMA(b) runs
//     wait MMA(b); load the norms of batch b+2 (cp.async build: also copy
//       rows(b+2) into the freed buffer, SW128 K-major layout)
//     row scans of b (tcgen05.ld); keys of b and their targets' loads
#pragma once
#include <climits>


#include "join_ws.cuh"

namespace knng {

constexpr int kTcRows = 128;     // sample slots per batch = MMA M = N
constexpr int kTcRowBytes = 128;  // bytes per staged row (uint8 rows of d <= 128)
constexpr int kTcWarps = 5;      // 4 epilogue/gather + 1 planning
constexpr int kTcThreads = kTcWarps * 32;
constexpr int kTcPlanWarp = 4;
constexpr int kTcCtasPerSm = 4;  // 4 x 128 TMEM columns
// TC_PGATHER: the planning warp issues the TMA row gathers of each batch
// (after the MMA two batches back has released the row buffer, signalled by
// a second tcgen05.commit) instead of 4 lanes of every epilogue warp
#ifndef TC_PGATHER
#define TC_PGATHER 1
#endif
#ifdef KNNG_TC_LOCKSTEP
#undef TC_PGATHER
#define TC_PGATHER 0
#endif
#ifndef TC_PMIN
#define TC_PMIN 1
#endif
#ifndef TC_PLANS
#define TC_PLANS 4
#endif
constexpr int kTcPlans = TC_PLANS;  // plan ring: b (scan), b+1, b+2 (rows in flight), b+3.. (being formed)

struct TcPlan {
    int nnodes;  // 0 = no more work
    int nslots;
    int sb[kWsMaxNodes], m[kWsMaxNodes], q[kWsMaxNodes];
    uint8_t map[kTcRows];  // slot -> node of the batch (0xFF: unused)
    uint32_t ids[kTcRows];
};

struct TcCfg {
    static constexpr size_t kRowBytes = static_cast<size_t>(kTcRows) * 128;  // one batch, SW128 K-major
    static constexpr size_t kNrmOff = 2 * kRowBytes;                           // int32 n'_c [3][128]
    static constexpr size_t kSideOff = kNrmOff + 3 * kTcRows * 4;              // u32 [3][4]
    static constexpr size_t kPlanOff = kSideOff + 3 * 4 * 4;
    static constexpr size_t kCacheOff = (kPlanOff + kTcPlans * sizeof(TcPlan) + 15) & ~size_t(15);
    static constexpr size_t kCacheCnt = 2 * 64;
    static constexpr size_t kCacheBytes = kCacheCnt + 2 * 32 * 2 * 32 * sizeof(uint32_t);
    static constexpr size_t kBarOff = (kCacheOff + kCacheBytes + 7) & ~size_t(7);
    static constexpr size_t kCombOff = (kBarOff + 8 * (1 + 2 * kTcPlans + 4) + 8 + 15) & ~size_t(15);
    static constexpr size_t kUsed = kCombOff + 2 * kTcRows * 4;  // + upper-half partial minima (EPI = 8)
    static constexpr size_t kSmem = kUsed + 1024;  // + slack to align the rows to 1024 B
    static_assert((kTcPlans > 4 ? 3 : kTcCtasPerSm) * (kSmem + 1024) <= 233472, "CTAs per SM");
};

// SW128 K-major shared-memory matrix descriptor (tcgen05): rows of 128 B,
// 8-row groups 1024 B apart, 16-B chunk c of row r stored at chunk c ^ (r & 7)
__device__ __forceinline__ uint64_t tc_smem_desc(uint32_t saddr) {
    return static_cast<uint64_t>((saddr >> 4) & 0x3FFF) | (1ull << 16) | (64ull << 32) | (1ull << 46) |
           (2ull << 61);
}
// instruction descriptor: kind::i8, u8 x u8 -> s32, K-major A and B, M = N = 128
constexpr uint32_t kTcIdesc = (2u << 4) | (0u << 7) | (0u << 10) | ((128u >> 3) << 17) | ((128u >> 4) << 24);

__device__ __forceinline__ void tc_mma_i8(uint32_t tmem, uint64_t ad, uint64_t bd, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
        "l"(ad), "l"(bd), "r"(kTcIdesc), "r"(accumulate));
}
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_ld16(uint32_t taddr, uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
// wait with the hardware suspend hint: the waiting warp is descheduled
// instead of polling (the planning warp is usually a full ring ahead)
__device__ __forceinline__ void mbar_wait_suspend(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity), "r"(1000000)
        : "memory");
}
// 0xFFFFFFFF << sh with the PTX clamp (sh >= 32 -> 0; unsigned, so a
// negative amount also gives 0)
__device__ __forceinline__ uint32_t shl_ones(uint32_t sh) {
    uint32_t r;
    asm("shl.b32 %0, %1, %2;" : "=r"(r) : "r"(0xFFFFFFFFu), "r"(sh));
    return r;
}
__device__ __forceinline__ uint32_t shl_clamp(uint32_t x, uint32_t sh) {
    uint32_t r;
    asm("shl.b32 %0, %1, %2;" : "=r"(r) : "r"(x), "r"(sh));
    return r;
}
// bits [a, b) of a 32-bit word for a <= b (a, b any ints): two clamped
// shifts, no branches
__device__ __forceinline__ uint32_t bit_range_fast(int a, int b) {
    return shl_ones(static_cast<uint32_t>(max(a, 0))) & ~shl_ones(static_cast<uint32_t>(max(b, 0)));
}
// bits [a, b) of a 32-bit word, clamped
__device__ __forceinline__ uint32_t bit_range(int a, int b) {
    a = max(a, 0);
    b = min(b, 32);
    if (a >= b) return 0u;
    const uint32_t hi = b >= 32 ? 0xFFFFFFFFu : ((1u << b) - 1u);
    return hi & ~((1u << a) - 1u);
}

// EPI epilogue warps: 4 (one thread per row), or 8 -- warps w and w + 4 read
// the same TMEM lane quarter and split the row's column chunks, the upper
// half handing its partial minima over through shared memory; 3 CTAs per SM
// then keep 24 epilogue warps resident instead of 16.
// TMA: rows gathered by TMA gather4 (one instruction per 4 rows, issued by
// the planning warp) instead of 16-B cp.async copies by every thread.
// REC: record mode of the distributed refine (dist_kernels.cuh) -- a template
// parameter, so the single-GPU build carries no per-key mode branch (the
// runtime check cost ~10 % of this kernel: 2.47 -> 2.73 ms per C2 launch).
template <int EPI, int CTAS, bool TMA, bool REC>
__global__ void __launch_bounds__((EPI + 1) * 32, CTAS)
k_join_tc(const uint8_t* __restrict__ X, const int* __restrict__ sqn, Dims D, Graph G, Samples S, int64_t boundary,
          unsigned long long* __restrict__ work, DevStats* __restrict__ stats,
          const __grid_constant__ CUtensorMap tmap) {
    static_assert(!TMA || EPI == 8, "the TMA gather spreads 32 row groups over 8 warps x 4 lanes");
    extern __shared__ __align__(16) unsigned char tc_raw[];
    // rows need 1024-B alignment (SW128 atoms)
    unsigned char* tc_smem = tc_raw + ((1024 - (smem_u32(tc_raw) & 1023)) & 1023);
    uint8_t* rows = tc_smem;
    int* nrm = reinterpret_cast<int*>(tc_smem + TcCfg::kNrmOff);
    uint32_t* side = reinterpret_cast<uint32_t*>(tc_smem + TcCfg::kSideOff);
    TcPlan* plans = reinterpret_cast<TcPlan*>(tc_smem + TcCfg::kPlanOff);
    uint8_t* cc_cnt = tc_smem + TcCfg::kCacheOff;
    uint32_t* cc_ids = reinterpret_cast<uint32_t*>(tc_smem + TcCfg::kCacheOff + TcCfg::kCacheCnt);
    uint64_t* mma_bar = reinterpret_cast<uint64_t*>(tc_smem + TcCfg::kBarOff);
    uint64_t* plan_full = mma_bar + 1;             // [kTcPlans] planning warp -> warps 0-3
    uint64_t* plan_empty = plan_full + kTcPlans;   // [kTcPlans] warps 0-3 -> planning warp
    uint64_t* rows_full = plan_empty + kTcPlans;  // [2] TMA row gathers of buffer 0 / 1
    uint64_t* rows_free = rows_full + 2;          // [2] MMA done reading buffer 0 / 1 (TC_PGATHER)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(rows_free + 2);
    int* comb = reinterpret_cast<int*>(tc_smem + TcCfg::kCombOff);
    constexpr int PW = EPI;  // the planning warp

    const int tid = threadIdx.x;
    const int warp = tid >> 5;
    const uint32_t lane = lane_id();
    const bool upper = tid >= kTcRows;  // EPI = 8: second half of the row's columns
    const int d = D.d, cap = D.cap;
    const bool restricted = boundary >= 0;
    const int kch = (d + 31) >> 5;  // MMAs of K = 32 (d % 16 == 0; zero-filled to 32)

    // ---------------------------------------------------------------- plans
    int cbuf = 1;
    uint32_t pend = 0;
    int64_t xnext = 0;
    unsigned long long claimed = 0;
    int my_m = 0, my_q = 0;
    bool more = true;
    unsigned long long n_joins = 0, n_m = 0, n_q = 0, n_rows = 0;  // n_rows: sample rows staged
    auto claim = [&]() -> unsigned long long {
        unsigned long long c0 = 0;
        if (lane == 0) c0 = atomicAdd(work, 32ull);
        return c0;
    };
    auto fetch = [&](int buf, int64_t xb) {
        if (xb < D.n) {
            const int nodes = static_cast<int>(D.n - xb < 32 ? D.n - xb : 32);
            const int64_t xl = xb + lane;
            if (lane < 16) {
                const int lo = 4 * static_cast<int>(lane), bytes = max(0, min(4, 2 * nodes - lo));
                asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(smem_u32(cc_cnt + buf * 64 + lo)),
                             "l"(S.gcnt + 2 * xb + lo), "r"(bytes)
                             : "memory");
            }
            uint32_t* cids = cc_ids + static_cast<size_t>(buf) * 32 * 2 * cap;
            if ((cap & 3) == 0) {
                if (static_cast<int>(lane) < nodes) {
                    const uint32_t* gn = S.G + static_cast<size_t>(xl) * cap;
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
    // the planning warp issues no other cp.async: its newest group is the
    // chunk it is about to use
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
        if (my_m > 0) {  // the join counters keep the method's m and q
            ++n_joins;
            n_m += my_m;
            n_q += my_q;
        }
        if (restricted && my_m > 0) {
            // GGM refine (D22): every NEW sample is cross-subset, so the only
            // pairs left are (NEW, OLD in x's own subset); OLD samples of the
            // other subset meet nothing.  Keep only the own-subset OLD ids
            // (in place, id order kept) -- fewer rows staged and scanned, and
            // a node without any is skipped.  Same candidates, same counts.
            uint32_t* orow = cc_ids + static_cast<size_t>(cbuf) * 32 * 2 * cap + lane * 2 * cap + cap;
            const bool xs = D.base + xnext + static_cast<int64_t>(lane) >= boundary;
            int qq = 0;
            for (int j = 0; j < my_q; ++j) {
                const uint32_t id = orow[j];
                if ((static_cast<int64_t>(id) >= boundary) == xs) orow[qq++] = id;
            }
            my_q = qq;
            if (qq == 0) my_m = 0;
        }
        pend = __ballot_sync(kFull, my_m > 0);
        xnext = static_cast<int64_t>(__shfl_sync(kFull, claimed, 0));
        claimed = claim();
        fetch(cbuf ^ 1, xnext);
        return true;
    };
    // first fit of whole nodes (m + q rows: NEW then OLD) into the 128 rows
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
                n_rows += m + q;
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
    // thread t (< 128) copies 16-B chunk (t & 7) of slots (t >> 3) + 16 i into
    // the SW128 layout; chunks in [d/16, 2 kch) are zero-filled
    const int part = tid & 7, row0 = tid >> 3;
    const int nchunks = d >> 4, kchunks = 2 * kch;
    int nv_next = 0, nv_prev = 0;  // this thread's slot norm of batches b+2 and b+1
    uint32_t side_next = 0, side_prev = 0;
    auto gather = [&](const TcPlan& P, uint8_t* dst) {
        const int nslots = P.nslots;  // hoisted: the asm below clobbers memory
        const uint32_t dbase = smem_u32(dst);
        if constexpr (TMA && TC_PGATHER) {
            // (rows issued by the planning warp)
        } else if constexpr (TMA) {
            // group g of 4 slots is issued by lane g % 4 of warp g / 4 (the
            // tx count may run ahead of the expect_tx: it is signed)
            const int ng = (nslots + 3) >> 2;  // groups of 4 slots; the tail repeats a valid row
            uint64_t* bar = rows_full + (dst == rows ? 0 : 1);
            if (tid == 0) mbar_expect_tx(bar, static_cast<uint32_t>(ng) * 512u);
            const int g = 4 * warp + static_cast<int>(lane);
            if (lane < 4 && warp < EPI) {
                if (g < ng) {
                    const int s0 = 4 * g;
                    const int r0 = static_cast<int>(P.ids[s0]);
                    const int r1 = s0 + 1 < nslots ? static_cast<int>(P.ids[s0 + 1]) : r0;
                    const int r2 = s0 + 2 < nslots ? static_cast<int>(P.ids[s0 + 2]) : r0;
                    const int r3 = s0 + 3 < nslots ? static_cast<int>(P.ids[s0 + 3]) : r0;
                    tma_gather4(dst + s0 * 128, &tmap, r0, r1, r2, r3, bar);
                }
            }
        } else if (part < nchunks) {
            const uint8_t* src0 = X + part * 16;
            for (int slot = row0; slot < nslots; slot += EPI * 4) {
                const uint32_t id = P.ids[slot];
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(
                                 dbase + slot * 128 + ((part ^ (slot & 7)) << 4)),
                             "l"(src0 + static_cast<size_t>(id) * d)
                             : "memory");
            }
        } else if (part < kchunks) {  // (cp.async path) chunks past d: zero-filled
            for (int slot = row0; slot < nslots; slot += EPI * 4)
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16, 0;\n" ::"r"(
                                 dbase + slot * 128 + ((part ^ (slot & 7)) << 4)),
                             "l"(X)
                             : "memory");
        }
        cp_async_commit();
        // squared norm of slot tid's row (exact integer), staged as n * 128 + slot
        if (!upper) {
            const uint32_t id = P.ids[tid];
            nv_next = id != 0xFFFFFFFFu ? __ldg(sqn + id) : 0;
            side_next = __ballot_sync(kFull, id != 0xFFFFFFFFu && static_cast<int64_t>(id) >= boundary);
        }
    };

    // --------------------------------------------------------------- filing
    // stage 1 (batch b): the row's 2 keys, its target (the row's sample) and
    // the target's k-th key / bucket offset loads; stage 2 (b+1): atomicAdd
    // slots; stage 3 (b+2): stores
    uint64_t f1_key[2], f1_th = 0, f1_bo = 0;
    uint32_t f1_tgt = 0;
    uint64_t f2_key[2], f2_pos[2];
    uint32_t f2_tgt = 0;
    // bucket mode: the slot returned by the count atomic is consumed only by
    // the next iteration's stores, so the atomic's return latency is not
    // waited for inside the iteration that issued it
    uint64_t f2_bo = 0;
    uint32_t f2_sl = 0, f2_ok0 = 0;
#pragma unroll
    for (int r = 0; r < 2; ++r) {
        f1_key[r] = kSentinel;
        f2_key[r] = kSentinel;
        f2_pos[r] = 0;
    }
    unsigned long long n_cand = 0, n_app = 0, my_pairs = 0;
    auto file_store = [&]() {
        if constexpr (REC) {  // record mode (distributed refine)
#pragma unroll
            for (int r = 0; r < 2; ++r)
                if (f2_key[r] != kSentinel) {
                    G.rec_key[f2_pos[r]] = f2_key[r];
                    G.rec_tgt[f2_pos[r]] = f2_tgt;
                }
        } else {
            const uint64_t p0 = f2_bo + f2_sl;
            if (f2_key[0] != kSentinel) G.bucket[p0] = f2_key[0];
            if (f2_key[1] != kSentinel) G.bucket[p0 + f2_ok0] = f2_key[1];
        }
    };
    auto file_atomic = [&]() {
        const bool ok0 = f1_key[0] < f1_th, ok1 = f1_key[1] < f1_th;  // D17 (the sentinel never passes)
        n_app += ok0 + ok1;
        if constexpr (REC) {
            // record slots: one atomic per warp (the call is warp-uniform)
            const uint32_t b0 = __ballot_sync(kFull, ok0), b1 = __ballot_sync(kFull, ok1);
            unsigned long long wb = 0;
            if (lane == 0 && (b0 | b1)) wb = atomicAdd(G.rec_cnt, static_cast<unsigned long long>(__popc(b0) + __popc(b1)));
            const uint64_t sl = shfl_u64(wb, 0) + __popc(b0 & lanemask_lt()) + __popc(b1 & lanemask_lt());
            f2_tgt = f1_tgt;
            f2_pos[0] = sl;
            f2_pos[1] = sl + (ok0 ? 1 : 0);
        } else {
            f2_sl = (ok0 || ok1) ? atomicAdd(G.bcnt + f1_tgt, static_cast<uint32_t>(ok0 + ok1)) : 0u;
            f2_bo = f1_bo;
            f2_ok0 = ok0 ? 1u : 0u;
        }
        f2_key[0] = ok0 ? f1_key[0] : kSentinel;
        f2_key[1] = ok1 ? f1_key[1] : kSentinel;
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
        mbar_init(rows_full, 1);
        mbar_init(rows_full + 1, 1);
        mbar_init(rows_free, 1);
        mbar_init(rows_free + 1, 1);
        for (int i = 0; i < kTcPlans; ++i) {
            mbar_init(plan_full + i, 1);
            mbar_init(plan_empty + i, PW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == PW) {
        // ---- planning warp: runs up to kTcPlans batches ahead
        xnext = static_cast<int64_t>(__shfl_sync(kFull, claim(), 0));
        claimed = claim();
        fetch(0, xnext);
#ifndef KNNG_TC_LOCKSTEP
        for (uint32_t t = 0;; ++t) {
            const int slot = t % kTcPlans;
            if (t >= kTcPlans) mbar_wait_suspend(plan_empty + slot, ((t / kTcPlans) - 1) & 1);
            form_plan(plans[slot]);
            const bool last = plans[slot].nnodes == 0;
            if (lane == 0) mbar_arrive(plan_full + slot);
            if (last) break;
            if constexpr (TMA && TC_PGATHER) {
                // rows of batch t into buffer t & 1 once MMA(t-2) has read it
                const int rb = t & 1;
                if (t >= 2) mbar_wait_suspend(rows_free + rb, ((t - 2) >> 1) & 1);
                const TcPlan& P = plans[slot];
                const int nslots = P.nslots, ng = (nslots + 3) >> 2;
                uint64_t* bar = rows_full + rb;
                if (lane == 0) mbar_expect_tx(bar, static_cast<uint32_t>(ng) * 512u);
                if (static_cast<int>(lane) < ng) {
                    const int s0 = 4 * static_cast<int>(lane);
                    const int r0 = static_cast<int>(P.ids[s0]);
                    const int r1 = s0 + 1 < nslots ? static_cast<int>(P.ids[s0 + 1]) : r0;
                    const int r2 = s0 + 2 < nslots ? static_cast<int>(P.ids[s0 + 2]) : r0;
                    const int r3 = s0 + 3 < nslots ? static_cast<int>(P.ids[s0 + 3]) : r0;
                    tma_gather4(rows + rb * TcCfg::kRowBytes + s0 * 128, &tmap, r0, r1, r2, r3, bar);
                }
            }
        }
#else
        // racecheck build (tools/racecheck_tc.sh): the same plans, but the
        // planning warp also meets the epilogue warps at a CTA barrier once
        // per batch (plan b+3 formed in iteration b), an ordering the race
        // checker models -- the default build orders the same hand-offs
        // with the plan_full / plan_empty mbarriers only
        uint32_t last_t = 0xFFFFFFFFu;
        auto form = [&](uint32_t t) {
            const int slot = t % kTcPlans;
            if (t >= kTcPlans) mbar_wait_suspend(plan_empty + slot, ((t / kTcPlans) - 1) & 1);
            if (last_t == 0xFFFFFFFFu) {
                form_plan(plans[slot]);
                if (plans[slot].nnodes == 0) last_t = t;
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(plan_full + slot);
        };
        for (uint32_t t = 0; t < 3; ++t) form(t);
        named_bar(6, (PW + 1) * 32);
        for (uint32_t b = 0; b < last_t; ++b) {
            if (b + 3 <= last_t) form(b + 3);
            named_bar(6, (PW + 1) * 32);
        }
#endif
    } else {
        // ---- warps 0-3: two batches of rows in flight
        bool ended = false;  // a terminator plan has been seen
#ifdef KNNG_TC_LOCKSTEP
        named_bar(6, (PW + 1) * 32);  // plans 0-2 formed
#endif
        for (int t = 0; t < 2; ++t) {
            if (!ended) {
                mbar_wait(plan_full + t, 0);
                ended = plans[t].nnodes == 0;
            }
            if (!ended) {
                gather(plans[t], rows + t * TcCfg::kRowBytes);
            } else {
                cp_async_commit();
            }
            if (t == 0) {
                if (!upper) {
                    nrm[tid] = nv_next * 128 + tid;
                    if (lane == 0) side[warp] = side_next;
                }
            } else {
                nv_prev = nv_next;
                side_prev = side_next;
            }
        }
        uint32_t b = 0;
        for (;; ++b) {
            const int slot = b % kTcPlans;
            const TcPlan& P = plans[slot];
            const int buf = b & 1;
            if (P.nnodes == 0) break;  // waited for at b - 2 (or in the prologue)
            if constexpr (!TMA) {
                cp_async_wait<1>();    // rows(b); rows(b+1) may be in flight
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // cp.async data -> MMA operand reads
            }
            named_bar(1, PW * 32);  // rows(b), n'(b) visible; TMEM reads of b-1 done
            if (tid == 0) {
                if constexpr (TMA) mbar_wait(rows_full + buf, (b >> 1) & 1);  // TMA rows(b) landed
                tc_fence_after();
                const uint32_t base = smem_u32(rows + buf * TcCfg::kRowBytes);
                for (int k = 0; k < kch; ++k) {
                    const uint64_t desc = tc_smem_desc(base + 32 * k);
                    tc_mma_i8(tmem, desc, desc, k > 0 ? 1u : 0u);
                }
                tc_commit(mma_bar);
                if constexpr (TMA && TC_PGATHER) tc_commit(rows_free + buf);
            }

            // ---- my row of batch b
            const int s = tid & (kTcRows - 1);
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
            // row masks as ranges: A = [alo, ahi) (the node's NEW columns,
            // scanned by NEW and OLD rows), B = [blo, bhi) (its OLD columns,
            // NEW rows only); empty ranges have lo = hi
            const int alo = act ? sb : 0, ahi = act ? sb + m : 0;
            const int blo = isNEW ? sb + m : 0, bhi = isNEW ? sb + m + q : 0;
            const uint32_t selfbit = isNEW ? 1u : 0u;
            // distance evaluations of the method (m(m-1)/2 + m q per join):
            // the NEW row of rank i pairs with the i NEW rows before it and
            // the q OLD rows -- closed form unless a GGM refine masks pairs
            if (!restricted && isNEW && !upper) my_pairs += (s - sb) + q;
            const uint32_t my_id = P.ids[s];
            const bool myside = restricted && static_cast<int64_t>(my_id) >= boundary;
            const int nbuf = b % 3;  // norms/sides: b (scan), b+1, b+2 (staged by other warps meanwhile)
            const int* nb = nrm + nbuf * kTcRows;
            const int ns = nb[s] >> 7;  // n_s
            int minA = INT_MAX, minB = INT_MAX;
            // deferred filing of the two previous batches while MMA(b) runs
            if (!upper) {
                file_store();
                file_atomic();
            }
            mbar_wait(mma_bar, b & 1);
            tc_fence_after();

            // ---- MMA(b) has read rows[buf]: gather batch b+2 into it
            if (!ended) {
                const int s2 = (b + 2) % kTcPlans;
#ifdef TC_SUSPEND
                mbar_wait_suspend(plan_full + s2, ((b + 2) / kTcPlans) & 1);
#else
                mbar_wait(plan_full + s2, ((b + 2) / kTcPlans) & 1);
#endif
                ended = plans[s2].nnodes == 0;
            }
            if (!ended) gather(plans[(b + 2) % kTcPlans], rows + buf * TcCfg::kRowBytes);
            else cp_async_commit();

            // 16-column chunks over the warp's column range (the union of its
            // rows' node ranges); EPI = 8 splits them between warps w, w + 4
            const int c0 = wlo & ~15;
            const int nchk = whi > c0 ? (whi - c0 + 15) >> 4 : 0;
            const int half = EPI == 8 ? (nchk + 1) >> 1 : nchk;
            const int cs = upper ? c0 + 16 * half : c0;
            const int ce = upper ? whi : min(whi, c0 + 16 * half);
            for (int cb = cs; cb < ce; cb += 16) {
                uint32_t A = bit_range_fast(alo - cb, ahi - cb) & ~shl_clamp(selfbit, static_cast<uint32_t>(s - cb));
                uint32_t B = bit_range_fast(blo - cb, bhi - cb);
                if (restricted) {
                    const uint32_t sd = side[nbuf * 4 + (cb >> 5)] >> (cb & 16);
                    const uint32_t allow = myside ? ~sd : sd;
                    A &= allow;
                    B &= allow;
                    // a GGM refine leaves whole chunks without a cross pair
                    // (NEW x NEW is always same-subset, D22): skip their loads
                    if (!__any_sync(kFull, ((A | B) & 0xFFFFu) != 0u)) continue;
                }
                uint32_t r[16];
                tc_ld16(tmem + (static_cast<uint32_t>((warp & 3) * 32) << 16) + cb, r);
                A &= 0xFFFFu;
                B &= 0xFFFFu;
                if (restricted && isNEW) my_pairs += __popc(A & ~shl_ones(static_cast<uint32_t>(max(s - cb, 0)))) + __popc(B);
                const int4* nv4 = reinterpret_cast<const int4*>(nb + cb);
                int kk[16];
#pragma unroll
                for (int g = 0; g < 4; ++g) {
                    const int4 n4 = nv4[g];
                    kk[4 * g] = n4.x - static_cast<int>(r[4 * g] << 8);
                    kk[4 * g + 1] = n4.y - static_cast<int>(r[4 * g + 1] << 8);
                    kk[4 * g + 2] = n4.z - static_cast<int>(r[4 * g + 2] << 8);
                    kk[4 * g + 3] = n4.w - static_cast<int>(r[4 * g + 3] << 8);
                }
                // masked minima, 3-input VIMNMX3; a mask that is empty on
                // every lane of the warp (OLD rows, chunks outside the OLD
                // range) is skipped as a whole
#if TC_PMIN
                // predicated minima (one IMNMX per selected element, the
                // predicates unpacked from the mask by R2P), two chains
                if (__any_sync(kFull, A != 0u)) {
                    int a1 = INT_MAX;
#pragma unroll
                    for (int e = 0; e < 16; e += 2) {
                        if ((A >> e) & 1u) minA = min(minA, kk[e]);
                        if ((A >> (e + 1)) & 1u) a1 = min(a1, kk[e + 1]);
                    }
                    minA = min(minA, a1);
                }
                if (__any_sync(kFull, B != 0u)) {
                    int b1 = INT_MAX;
#pragma unroll
                    for (int e = 0; e < 16; e += 2) {
                        if ((B >> e) & 1u) minB = min(minB, kk[e]);
                        if ((B >> (e + 1)) & 1u) b1 = min(b1, kk[e + 1]);
                    }
                    minB = min(minB, b1);
                }
#else
                if (__any_sync(kFull, A != 0u)) {
#pragma unroll
                    for (int e = 0; e < 16; e += 2)
                        minA = __vimin3_s32(minA, (A >> e) & 1u ? kk[e] : INT_MAX,
                                            (A >> (e + 1)) & 1u ? kk[e + 1] : INT_MAX);
                }
                if (__any_sync(kFull, B != 0u)) {
#pragma unroll
                    for (int e = 0; e < 16; e += 2)
                        minB = __vimin3_s32(minB, (B >> e) & 1u ? kk[e] : INT_MAX,
                                            (B >> (e + 1)) & 1u ? kk[e + 1] : INT_MAX);
                }
#endif
            }
            tc_fence_before();
            if constexpr (EPI == 8) {
                if (upper) {
                    comb[s] = minA;
                    comb[kTcRows + s] = minB;
                }
                named_bar(2 + (warp & 3), 64);  // the pair (w, w + 4) only
                if (!upper) {
                    minA = min(minA, comb[s]);
                    minB = min(minB, comb[kTcRows + s]);
                }
            }

            // ---- this batch's keys (filed in iterations b+1 and b+2)
            uint64_t k1 = kSentinel, k2 = kSentinel;
            if (!upper && act && minA != INT_MAX)
                k1 = make_key(static_cast<float>(ns + (minA >> 7)), P.ids[minA & 127]);
            if (!upper && isNEW && minB != INT_MAX)
                k2 = make_key(static_cast<float>(ns + (minB >> 7)), P.ids[minB & 127]);
            f1_key[0] = k1;
            f1_key[1] = k2;
            f1_tgt = my_id;
            n_cand += (k1 != kSentinel) + (k2 != kSentinel);
            if (k1 != kSentinel || k2 != kSentinel) {  // D15: (inf, inf) inserts nothing
                f1_th = __ldg(G.kth_t + my_id);
                if constexpr (!REC) f1_bo = __ldg(G.boff + my_id);
            }
            // batch b+1's norms (their loads were issued one iteration ago);
            // buffer (b+1) % 3 was last read by the scans of b-2
            __syncwarp();
            if (!upper) nrm[((b + 1) % 3) * kTcRows + tid] = nv_prev * 128 + tid;
            nv_prev = nv_next;
            if (lane == 0) {
                if (!upper) side[((b + 1) % 3) * 4 + warp] = side_prev;
                mbar_arrive(plan_empty + slot);  // this warp is done with plan b
            }
            side_prev = side_next;
#ifdef KNNG_TC_LOCKSTEP
            named_bar(6, (PW + 1) * 32);
#endif
        }
        if constexpr (TMA && TC_PGATHER) {
            // the row-buffer releases of the last two batches have landed
            // before the shared memory goes away
            if (tid == 0)
                for (uint32_t l = b > 2 ? b - 2 : 0; l < b; ++l) mbar_wait(rows_free + (l & 1), (l >> 1) & 1);
        }
    }
    if (warp < PW && !upper) {
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
        n_rows += __shfl_xor_sync(kFull, n_rows, o);
    }
    if (lane == 0) {
        if (n_cand) atomicAdd(&stats->candidates, n_cand);
        if (n_app) atomicAdd(&stats->appended, n_app);
        if (my_pairs) atomicAdd(&stats->dist_evals, my_pairs);
        if (warp == PW && n_joins) {
            atomicAdd(&stats->joins, n_joins);
            atomicAdd(&stats->sum_m, n_m);
            atomicAdd(&stats->sum_q, n_q);
            atomicAdd(&stats->rows, n_rows);
        }
    }
}

// exact squared norms of uint8 rows (int32; d <= 128 keeps them < 2^23);
// d % 16 == 0 and 16-B aligned rows (the tensor-core join's preconditions)
__global__ void k_sqnorm_u8(const uint8_t* __restrict__ X, int64_t n, int d, int* __restrict__ out) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint4* x = reinterpret_cast<const uint4*>(X + i * d);
    unsigned int acc = 0;
    for (int j = 0; j < d / 16; ++j) {
        const uint4 v = __ldg(x + j);
        acc = __dp4a(v.x, v.x, acc);
        acc = __dp4a(v.y, v.y, acc);
        acc = __dp4a(v.z, v.z, acc);
        acc = __dp4a(v.w, v.w, acc);
    }
    out[i] = static_cast<int>(acc);
}

}  // namespace knng
