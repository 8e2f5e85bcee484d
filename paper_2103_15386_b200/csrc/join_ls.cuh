// join_ls.cuh -- lock-step local join for uint8 rows of <= 128 dims
// (Alg. 1 lines 9-31; the exact-u8 path of D35).
//
// Same computation and outputs as k_join_ws (join_ws.cuh), organised for the
// case where one 128-B row slab holds a whole sample row: every batch is a
// single ring stage, so the warp-specialised pipeline spent most of its issue
// slots on mbarrier hand-offs (profiles/r01_ncu_join_v21.txt: 41% issue
// active, 23% of it distance arithmetic).  Here every warp of the CTA runs
// every phase, two CTAs per SM hide each other's barriers, and the
// three-level dependency chain (chunk -> batch plan -> rows) is software
// pipelined:
//
//   iteration b:  wait rows(b) ; sync
//                 issue cp.async rows(b+1)          (plan b+1 formed at b-1)
//                 tile(b): one 4x4 register block per thread -> partial minima
//                 sync
//                 file(b-2) stores, file(b-1) atomics   (deferred, see below)
//                 reduce(b): GetNearestObject per output key (Alg. 2), then
//                            issue the target loads of file(b)
//                 last warp: plan(b+2) from the chunk cache
//
// Plans: the last warp packs consecutive nodes of a 32-node chunk into a batch whose
// 4x4 blocks fit the 256 threads and whose sample rows fit the 256 slots.
// Chunks are claimed from a global counter two ahead; the next chunk's
// (m, q) counts and sample-id rows are prefetched with cp.async.
//
// Filing (the k_cand_scatter step, fused): key -> load the target's
// iteration-start k-th key and bucket offset -> atomicAdd on its bucket count
// -> store.  The three dependent global steps of batch b run in iterations
// b, b+1 and b+2, so their latency hides behind the tiles of later batches.
#pragma once
#include "join_ws.cuh"

namespace knng {

constexpr int kLsThreads = 256;
constexpr int kLsBlocks = 256;  // 4x4 blocks per batch, one per thread
constexpr int kLsSlots = 256;   // sample rows per batch
constexpr int kLsRow = 128;     // bytes per staged row (d <= 128 uint8)
constexpr int kLsKeys = 2;      // output keys per thread: sum(2m+q) <= 2 * slots
// the planning warp: the last one, whose threads most often own no block
// (blocks fill the batch from thread 0)
constexpr int kLsPlanWarp = kLsThreads / 32 - 1;

struct LsPlan {
    int nnodes;  // 0 = no more work
    int nblocks, nslots, nout;
    int m[kWsMaxNodes], q[kWsMaxNodes], sbase[kWsMaxNodes];
    int bbase[kWsMaxNodes + 1], obase[kWsMaxNodes + 1];
    uint32_t ids[kLsSlots];
};

struct LsCfg {
    static constexpr size_t kRowBytes = static_cast<size_t>(kLsSlots) * kLsRow;        // one batch
    static constexpr size_t kPartOff = 2 * kRowBytes;                                   // rows: double-buffered
    static constexpr size_t kPartBytes = sizeof(unsigned long long) * 8 * kLsBlocks;    // row + col minima
    static constexpr size_t kPlanOff = kPartOff + kPartBytes;
    static constexpr size_t kCacheOff = (kPlanOff + 3 * sizeof(LsPlan) + 15) & ~size_t(15);
    static constexpr size_t kCacheCnt = 2 * 64;                                         // (m, q) bytes
    static constexpr size_t kCacheBytes = kCacheCnt + 2 * 32 * 2 * 32 * sizeof(uint32_t);  // + id rows
    static constexpr size_t kSmem = kCacheOff + kCacheBytes;
    static_assert(2 * (kSmem + 1024) <= 233472, "two CTAs per SM");
};

__global__ void __launch_bounds__(kLsThreads, 2)
k_join_ls(const uint8_t* __restrict__ X, Dims D, Graph G, Samples S, int64_t boundary,
          unsigned long long* __restrict__ work, DevStats* __restrict__ stats) {
    extern __shared__ __align__(128) unsigned char ls_smem[];
    uint8_t* rows = ls_smem;
    unsigned long long* parts = reinterpret_cast<unsigned long long*>(ls_smem + LsCfg::kPartOff);
    LsPlan* plans = reinterpret_cast<LsPlan*>(ls_smem + LsCfg::kPlanOff);
    uint8_t* cc_cnt = ls_smem + LsCfg::kCacheOff;
    uint32_t* cc_ids = reinterpret_cast<uint32_t*>(ls_smem + LsCfg::kCacheOff + LsCfg::kCacheCnt);

    const int tid = threadIdx.x;
    const int warp = tid >> 5;
    const uint32_t lane = lane_id();
    const int d = D.d, cap = D.cap;
    const bool restricted = boundary >= 0;

    // ---------------------------------------------------------------- plans
    // planning-warp state: lane = node of the current chunk
    int cbuf = 1;
    uint32_t pend = 0;  // nodes of the current chunk not yet in a batch
    int64_t x0 = 0, xnext = 0;
    unsigned long long claimed = 0;
    int my_m = 0, my_q = 0, my_nb = 0, my_sl = 0;
    bool more = true;
    bool fetch_last = false;  // the newest cp.async group is a chunk prefetch
    unsigned long long n_joins = 0, n_m = 0, n_q = 0;
    auto claim = [&]() -> unsigned long long {
        unsigned long long c0 = 0;
        if (lane == 0) c0 = atomicAdd(work, 32ull);
        return c0;  // lane 0's value; broadcast at use
    };
    auto fetch = [&](int buf, int64_t xb) {
        if (xb < D.n) {
            const int nodes = static_cast<int>(D.n - xb < 32 ? D.n - xb : 32);
            if (lane < 16) {  // (m, q) byte pairs, 4 bytes per lane, zero-filled past n
                const int lo = 4 * static_cast<int>(lane), bytes = max(0, min(4, 2 * nodes - lo));
                asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(smem_u32(cc_cnt + buf * 64 + lo)),
                             "l"(S.gcnt + 2 * xb + lo), "r"(bytes)
                             : "memory");
            }
            uint32_t* cids = cc_ids + static_cast<size_t>(buf) * 32 * 2 * cap;
            if ((cap & 3) == 0) {  // rows of 16-B multiples: lane = node, 16-B copies
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
                cp_async_commit();
                fetch_last = true;
                return;
            }
            for (int e = lane; e < nodes * 2 * cap; e += 32) {
                const int node = e / (2 * cap), w = e - node * 2 * cap;
                const uint32_t* src = w < cap ? S.G + static_cast<size_t>(xb + node) * cap + w
                                              : S.G + static_cast<size_t>(D.n) * cap +
                                                    static_cast<size_t>(xb + node) * cap + (w - cap);
                asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(smem_u32(cids + e)), "l"(src)
                             : "memory");
            }
        }
        cp_async_commit();
        fetch_last = true;
    };
    // move to the prefetched chunk; false when the work is exhausted
    auto advance = [&]() -> bool {
        if (xnext >= D.n) return false;
        // the chunk's prefetch group is complete once at most the newest
        // group (a row gather issued after it) is pending
        if (fetch_last) cp_async_wait<0>();
        else cp_async_wait<1>();
        __syncwarp();
        cbuf ^= 1;
        x0 = xnext;
        my_m = 0;
        my_q = 0;
        if (x0 + lane < D.n) {
            my_m = cc_cnt[cbuf * 64 + 2 * lane];
            my_q = cc_cnt[cbuf * 64 + 2 * lane + 1];
        }
        if (my_m == 0) my_q = 0;  // no NEW sample: nothing to join
        const int mg = (my_m + 3) >> 2, qg = (my_q + 3) >> 2;
        my_nb = mg * (mg + 1) / 2 + mg * qg;
        my_sl = 4 * (mg + qg);
        pend = __ballot_sync(kFull, my_m > 0);
        xnext = static_cast<int64_t>(__shfl_sync(kFull, claimed, 0));
        claimed = claim();
        fetch(cbuf ^ 1, xnext);
        return true;
    };
    // first-fit packing: take pending nodes in chunk order, skipping any that
    // no longer fit, until no pending node fits the remaining blocks/slots
    // (node order inside a batch is free: every node's outputs are its own)
    auto form_plan = [&](LsPlan& P) {
        while (pend == 0) {
            if (!more || !advance()) {
                more = false;
                if (lane == 0) P.nnodes = 0;
                __syncwarp();  // the terminator is read by every lane
                return;
            }
        }
        const uint32_t* cids = cc_ids + static_cast<size_t>(cbuf) * 32 * 2 * cap;
        int nb_used = 0, ns_used = 0, no_used = 0, nn = 0;
        while (true) {
            const bool fit = ((pend >> lane) & 1u) && my_nb <= kLsBlocks - nb_used && my_sl <= kLsSlots - ns_used;
            const uint32_t fm = __ballot_sync(kFull, fit);
            if (fm == 0) break;
            const int L = __ffs(fm) - 1;
            const int m = __shfl_sync(kFull, my_m, L), q = __shfl_sync(kFull, my_q, L);
            if (static_cast<int>(lane) == L) {
                P.m[nn] = m;
                P.q[nn] = q;
                P.sbase[nn] = ns_used;
                P.bbase[nn] = nb_used;
                P.obase[nn] = no_used;
                ++n_joins;
                n_m += m;
                n_q += q;
            }
            // sample ids of the node's slots: [Gn, pad to 4, Go, pad to 4]
            const int mpad = (m + 3) & ~3, len = mpad + ((q + 3) & ~3);
            const uint32_t* row = cids + L * 2 * cap;
            for (int js = lane; js < len; js += 32) {
                uint32_t id = 0xFFFFFFFFu;
                if (js < m) id = row[js];
                else if (js >= mpad && js - mpad < q) id = row[cap + (js - mpad)];
                P.ids[ns_used + js] = id;
            }
            const int mg = mpad >> 2, qg = (q + 3) >> 2;
            nb_used += mg * (mg + 1) / 2 + mg * qg;
            ns_used += len;
            no_used += 2 * m + q;
            pend &= ~(1u << L);
            ++nn;
        }
        if (lane == 0) {
            P.nnodes = nn;
            P.nblocks = nb_used;
            P.nslots = ns_used;
            P.nout = no_used;
            P.bbase[nn] = nb_used;
            P.obase[nn] = no_used;
        }
        __syncwarp();
    };

    // ------------------------------------------------------------- gathers
    // thread t copies 16-B chunk (t & 7) of slots (t >> 3) + 32 i; chunks are
    // XOR-swizzled by (slot >> 2) & 7 (conflict-free LDS.128 in the tile)
    const int part = tid & 7, row0 = tid >> 3;
    const int nchunks = d >> 4;  // d % 16 == 0 (host check)
    auto gather = [&](const LsPlan& P, uint8_t* dst) {
        if (part < nchunks) {
            const uint8_t* src0 = X + part * 16;
            for (int slot = row0; slot < P.nslots; slot += kLsThreads / 8) {
                const uint32_t id = P.ids[slot];
                if (id == 0xFFFFFFFFu) continue;
                const int c = part ^ ((slot >> 2) & 7);
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(dst + slot * kLsRow + c * 16)),
                             "l"(src0 + static_cast<size_t>(id) * d)
                             : "memory");
            }
        }
        cp_async_commit();
        fetch_last = false;
    };

    // --------------------------------------------------------------- filing
    // stage 1 (batch b): key, target, loads of kth/boff; stage 2 (b+1):
    // atomicAdd slot; stage 3 (b+2): store
    uint64_t f1_key[kLsKeys], f1_th[kLsKeys], f1_bo[kLsKeys];
    uint32_t f1_tgt[kLsKeys];
    uint64_t f2_key[kLsKeys], f2_bo[kLsKeys];
    uint32_t f2_sl[kLsKeys];
#pragma unroll
    for (int r = 0; r < kLsKeys; ++r) {
        f1_key[r] = kSentinel;
        f1_th[r] = 0;
        f1_bo[r] = 0;
        f1_tgt[r] = 0;
        f2_key[r] = kSentinel;
        f2_bo[r] = 0;
        f2_sl[r] = 0xFFFFFFFFu;
    }
    unsigned long long n_cand = 0, n_app = 0, my_pairs = 0;
    auto file_store = [&]() {
#pragma unroll
        for (int r = 0; r < kLsKeys; ++r)
            if (f2_sl[r] != 0xFFFFFFFFu) G.bucket[f2_bo[r] + f2_sl[r]] = f2_key[r];
    };
    auto file_atomic = [&]() {  // stage 1 -> stage 2
#pragma unroll
        for (int r = 0; r < kLsKeys; ++r) {
            const bool ok = f1_key[r] != kSentinel && f1_key[r] < f1_th[r];  // D17
            n_app += ok;
            f2_sl[r] = ok ? atomicAdd(G.bcnt + f1_tgt[r], 1u) : 0xFFFFFFFFu;
            f2_key[r] = f1_key[r];
            f2_bo[r] = f1_bo[r];
            f1_key[r] = kSentinel;
        }
    };

    // ------------------------------------------------------------- prologue
    if (warp == kLsPlanWarp) {
        xnext = static_cast<int64_t>(__shfl_sync(kFull, claim(), 0));
        claimed = claim();
        fetch(0, xnext);
        form_plan(plans[0]);
        form_plan(plans[1]);
    }
    __syncthreads();
    if (plans[0].nnodes > 0) gather(plans[0], rows);

    for (uint32_t b = 0;; ++b) {
        const LsPlan& P = plans[b % 3];
        cp_async_wait<0>();
        __syncthreads();  // rows(b) and plan(b+1) visible
        if (P.nnodes == 0) break;
        {
            const LsPlan& Pn = plans[(b + 1) % 3];
            if (Pn.nnodes > 0) gather(Pn, rows + ((b + 1) & 1) * LsCfg::kRowBytes);
        }

        // ---- tile: my 4x4 block of the batch
        const int nn = P.nnodes;
        const int ct = tid;
        const bool active = ct < P.nblocks;
        int nd = 0;
        if (active)
            while (nd + 1 < nn && P.bbase[nd + 1] <= ct) ++nd;
        const int m = P.m[nd], q = P.q[nd], sb = P.sbase[nd];
        const int mpad = (m + 3) & ~3, mg = mpad >> 2, qg = (q + 3) >> 2;
        const int t = ct - P.bbase[nd];
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
        const int fA = ((sb + rb) >> 2) & 7, fB = ((sb + cb) >> 2) & 7;
        unsigned int acc[4][4];
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
            for (int c = 0; c < 4; ++c) acc[r][c] = 0u;
        if (active) {
            const uint8_t* A = rows + (b & 1) * LsCfg::kRowBytes + (sb + rb) * kLsRow;
            const uint8_t* B = rows + (b & 1) * LsCfg::kRowBytes + (sb + cb) * kLsRow;
            // exact integer sum of squares (D5): one LDS.128 per row brings
            // 16 dims, 2 instructions per 4 dims and pair
#pragma unroll 2
            for (int j = 0; j < 8; ++j) {
                if (j >= nchunks) break;
                uint4 a[4], bv[4];
#pragma unroll
                for (int r = 0; r < 4; ++r) a[r] = *reinterpret_cast<const uint4*>(A + r * kLsRow + ((j ^ fA) << 4));
#pragma unroll
                for (int c = 0; c < 4; ++c) bv[c] = *reinterpret_cast<const uint4*>(B + c * kLsRow + ((j ^ fB) << 4));
#pragma unroll
                for (int r = 0; r < 4; ++r)
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        uint32_t ad;
                        ad = __vabsdiffu4(a[r].x, bv[c].x); acc[r][c] = __dp4a(ad, ad, acc[r][c]);
                        ad = __vabsdiffu4(a[r].y, bv[c].y); acc[r][c] = __dp4a(ad, ad, acc[r][c]);
                        ad = __vabsdiffu4(a[r].z, bv[c].z); acc[r][c] = __dp4a(ad, ad, acc[r][c]);
                        ad = __vabsdiffu4(a[r].w, bv[c].w); acc[r][c] = __dp4a(ad, ad, acc[r][c]);
                    }
            }
            // block minima: 4 row keys (c_nn / c_no candidates of the NEW rows)
            // and 4 column keys (c_nn / c_on candidates of the columns)
            unsigned long long* rowp = parts;
            unsigned long long* colp = parts + 4 * kLsBlocks;
            const uint32_t* nid = P.ids + sb;
            uint32_t rid[4], cid[4];
#pragma unroll
            for (int r = 0; r < 4; ++r) rid[r] = nid[rb + r];
#pragma unroll
            for (int c = 0; c < 4; ++c) cid[c] = nid[cb + c];
            uint64_t colbest[4] = {kSentinel, kSentinel, kSentinel, kSentinel};
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const int u = rb + r;
                uint64_t rowbest = kSentinel;
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const int w = cb + c;
                    bool valid = nn_blk ? (u < m && w < u) : (u < m && (w - mpad) < q);
                    if (restricted && valid) valid = allowed_pair(boundary, rid[r], cid[c]);
                    if (!valid) continue;
                    const float dist = static_cast<float>(acc[r][c]);
                    ++my_pairs;
                    const uint64_t kr = make_key(dist, cid[c]);
                    const uint64_t kc = make_key(dist, rid[r]);
                    rowbest = kr < rowbest ? kr : rowbest;
                    colbest[c] = kc < colbest[c] ? kc : colbest[c];
                }
                rowp[ct * 4 + r] = rowbest;
            }
#pragma unroll
            for (int c = 0; c < 4; ++c) colp[ct * 4 + c] = colbest[c];
        }
        __syncthreads();  // partials complete

        // ---- deferred filing of the two previous batches
        file_store();
        file_atomic();

        // ---- GetNearestObject per output key (Alg. 2): output o is key j of
        // node i (obase[i] <= o): c_nn(u_j) (j < m), c_no(u_{j-m}) (j < 2m),
        // c_on(w_{j-2m}); the min over the partials of the blocks covering it
        const int total = P.nout;
#pragma unroll
        for (int r = 0; r < kLsKeys; ++r) {
            const int o = tid + r * kLsThreads;
            uint64_t v = kSentinel;
            uint32_t tgt = 0;
            if (o < total) {
                int i = 0;
                while (i + 1 < nn && P.obase[i + 1] <= o) ++i;
                const int j = o - P.obase[i];
                const int mi = P.m[i], qi = P.q[i];
                const int mgi = (mi + 3) >> 2, qgi = (qi + 3) >> 2, bb = P.bbase[i];
                const int nnn_i = mgi * (mgi + 1) / 2;
                // the partials covering the key form one or two strided runs
                // (in u64 units): run A of na entries from a0 step sa, then
                // (c_nn only) run B from b0 with a step growing by 4 each time
                int na, a0, sa, nb = 0, b0 = 0, sb0 = 0;
                if (j < mi) {  // c_nn(u): row of blocks (I, J <= I), column of (I' >= I, I)
                    const int Iu = j >> 2, rr = j & 3;
                    na = Iu + 1;
                    a0 = (bb + Iu * (Iu + 1) / 2) * 4 + rr;
                    sa = 4;
                    nb = mgi - Iu;
                    b0 = 4 * kLsBlocks + (bb + Iu * (Iu + 1) / 2 + Iu) * 4 + rr;
                    sb0 = 4 * (Iu + 1);
                } else if (j < 2 * mi) {  // c_no(u): rows of the NEW-OLD blocks (I, J)
                    const int u = j - mi, Iu = u >> 2, rr = u & 3;
                    na = qgi;
                    a0 = (bb + nnn_i + Iu * qgi) * 4 + rr;
                    sa = 4;
                } else {  // c_on(w): columns of the NEW-OLD blocks (I, J_w)
                    const int oo = j - 2 * mi;
                    na = mgi;
                    a0 = 4 * kLsBlocks + (bb + nnn_i + (oo >> 2)) * 4 + (oo & 3);
                    sa = 4 * qgi;
                }
                const int ntot = na + nb;
                int addr = a0, step = sa;
                for (int t = 0; t < ntot; ++t) {
                    if (t == na) {
                        addr = b0;
                        step = sb0;
                    }
                    const uint64_t tv = parts[addr];
                    v = tv < v ? tv : v;
                    addr += step;
                    if (t >= na) step += 4;
                }
                // target: the NEW sample u_j (c_nn, c_no) or the OLD sample w_j (c_on)
                const int sbi = P.sbase[i], mpi = (mi + 3) & ~3;
                tgt = P.ids[j < mi ? sbi + j : (j < 2 * mi ? sbi + j - mi : sbi + mpi + j - 2 * mi)];
            }
            f1_key[r] = v;
            f1_tgt[r] = tgt;
            f1_th[r] = 0;
            f1_bo[r] = 0;
            if (v != kSentinel) {  // D15: (inf, inf) inserts nothing
                ++n_cand;
                f1_th[r] = __ldg(G.kth + tgt);
                f1_bo[r] = __ldg(G.boff + tgt);
            }
        }

        // ---- the plan two batches ahead
        if (warp == kLsPlanWarp) form_plan(plans[(b + 2) % 3]);
    }
    // drain the filing pipeline
    file_store();
    file_atomic();
    file_store();
    cp_async_wait<0>();

#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        n_cand += __shfl_xor_sync(kFull, n_cand, o);
        n_app += __shfl_xor_sync(kFull, n_app, o);
        my_pairs += __shfl_xor_sync(kFull, my_pairs, o);
        n_joins += __shfl_xor_sync(kFull, n_joins, o);
        n_m += __shfl_xor_sync(kFull, n_m, o);
        n_q += __shfl_xor_sync(kFull, n_q, o);
    }
    if (lane == 0) {
        if (n_cand) atomicAdd(&stats->candidates, n_cand);
        if (n_app) atomicAdd(&stats->appended, n_app);
        if (my_pairs) atomicAdd(&stats->dist_evals, my_pairs);
        if (warp == kLsPlanWarp && n_joins) {
            atomicAdd(&stats->joins, n_joins);
            atomicAdd(&stats->sum_m, n_m);
            atomicAdd(&stats->sum_q, n_q);
            atomicAdd(&stats->rows, n_m + n_q);
        }
    }
}

}  // namespace knng
