// join_ws.cuh -- warp-specialised local join (Alg. 1 lines 9-31).
//
// Same computation as k_join (join_kernel.cuh), organised as a three-role
// pipeline for sm_100a (one persistent CTA per SM, 16 warps; the light roles
// on the highest warp ids, which the issue arbiter serves first):
//
//  producers (4 warps): the lead warp grabs chunks of 32 nodes from a global
//      work counter and packs consecutive nodes into a batch whose 4x4
//      register blocks fit the 256 consumer threads (one block each) and
//      whose sample rows fit one ring stage; it publishes the batch metadata
//      (node table, sample ids) into a kWsMeta-deep ring, running ahead of
//      the rest.  3 gather warps issue the 16-B cp.async copies of each
//      128-B row slab of the batch's rows into a STAGES-deep ring; each thread signals completion with
//      cp.async.mbarrier.arrive.noinc on the stage's full barrier.  (One
//      cp.async.bulk per 128-B row slab was tried first: those copies
//      serialise through uniform registers on the issuing warp, ~90 cycles
//      each, IPC 0.75 -- profiles/r01_ncu_join_v4.txt.)
//  consumers (8 warps): each thread owns one 4x4 block of the batch's tiles
//      (NEW rows x sample columns), accumulates the canonical distance
//      (D5/D6) slab by slab as the ring fills, releases each stage with one
//      arrive per warp, and leaves the block's 4 row minima and 4 column
//      minima (packed (d, id) keys, D3) in a double-buffered partials area.
//  epilogue (2 groups of 2 warps, alternate batches): GetNearestObject (Alg. 2) per output slot -- the min
//      over the partials of the blocks covering the sample (the paper's
//      atomicMin on (v, d), without atomics) -- and files the 2m+q
//      keys of every node into their targets' buckets (the k_cand_scatter
//      step, fused); then releases the partials and metadata.
//
// Consumers never wait for each other: the selection/output epilogue of
// batch b runs on its own warps while batch b+1 is computed, and the
// gathers of later batches stream into the ring meanwhile.
#pragma once
#include <cuda.h>  // CUtensorMap (the TMA descriptor type; no driver-API linking)

#include "join_kernel.cuh"

namespace knng {

constexpr int kWsConsumerWarps = 8;
constexpr int kWsProducerWarps = 8;  // 1 lead (batch metadata) + 7 gather warps
constexpr int kWsGatherWarps = kWsProducerWarps - 1;
constexpr int kWsEpiGroups = 2;      // epilogue groups, alternating batches
constexpr int kWsEpiGroupWarps = 2;
constexpr int kWsEpilogueWarps = kWsEpiGroups * kWsEpiGroupWarps;
constexpr int kWsProdThreads = kWsGatherWarps * 32;
constexpr int kWsEpiThreads = kWsEpiGroupWarps * 32;  // threads of one epilogue group
constexpr int kWsThreads = (kWsConsumerWarps + kWsProducerWarps + kWsEpilogueWarps) * 32;
constexpr int kWsSlots = 256;    // sample rows per stage (all nodes of a batch)
constexpr int kWsBlocks = kWsConsumerWarps * 32;  // 4x4 blocks per batch
constexpr int kWsMaxNodes = 32;  // nodes per batch (one producer chunk)
constexpr int kWsMeta = 3;
// selected keys per batch <= sum(2m + q) <= 2 * slots: rounds of the epilogue
constexpr int kEpiRounds = (2 * kWsSlots + kWsEpiThreads - 1) / kWsEpiThreads;
static_assert(kWsEpiGroups == 2, "partials are double-buffered: one buffer per epilogue group");

struct WsMeta {
    int nnodes;   // 0 = no more work
    int nblocks;
    int nslots;
    int pad_;
    int64_t x[kWsMaxNodes];
    int m[kWsMaxNodes], q[kWsMaxNodes], sbase[kWsMaxNodes], bbase[kWsMaxNodes + 1];
    int obase[kWsMaxNodes + 1];  // prefix of the 2m+q selected keys per node
    uint32_t ids[kWsSlots];
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
// Wait until the phase with the given parity has completed.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// Same, for the non-consumer roles: back off with nanosleep between polls.
// The warp arbiter favours the highest warp id (B300_MICROARCH.md), so the
// consumers sit on the high ids and everybody else polls politely.
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
    uint32_t done = 0, ns = 32;
    while (true) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
        if (done) return;
        __nanosleep(ns);
        ns = ns < 512 ? ns * 2 : 512;
    }
}
// Idle wait of the roles with slack (gather, lead, epilogue) in the packed
// join: test once, then plain nanosleep back-off (not woken by barrier
// traffic).  Every test is a shared-memory barrier operation competing with
// the consumers' LDS.  (try_wait with a suspend-time hint compiles to
// TRYWAIT + NANOSLEEP.SYNCS, which every arrive in the CTA wakes: under ncu
// SYNCS + NANOSLEEP + BRA were 46 % of the kernel's instructions.)
#ifndef WS_IDLE_MAX_NS
#define WS_IDLE_MAX_NS 1024
#endif
#ifndef WS_IDLE_MIN_NS
#define WS_IDLE_MIN_NS 64
#endif
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
    uint32_t done;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return done != 0;
}
__device__ __forceinline__ void mbar_wait_idle(uint64_t* bar, uint32_t parity) {
    uint32_t ns = WS_IDLE_MIN_NS;
    while (!mbar_test(bar, parity)) {
        __nanosleep(ns);
        ns = ns < WS_IDLE_MAX_NS ? 2 * ns : WS_IDLE_MAX_NS;
    }
}
// Packed FP32x2 steps of the canonical accumulation (D5/D6) for two pairs
// (a, b0) and (a, b1) at once: b = {b0_i, b1_i}, acc = {acc0, acc1}.  Both
// lanes are IEEE round-to-nearest sub and fused multiply-add, i.e. exactly
// t = a_i - b_i; acc = fmaf(t, t, acc) of each pair (FADD2 / FFMA2 on
// sm_100a, the scalar a broadcast by the .F32 operand selector).
__device__ __forceinline__ unsigned long long f2_l2(float a, unsigned long long b, unsigned long long acc) {
    unsigned long long r;
    asm("{\n\t.reg .b64 aa, tt;\n\tmov.b64 aa, {%1, %1};\n\tsub.rn.f32x2 tt, aa, %2;\n\t"
        "fma.rn.f32x2 %0, tt, tt, %3;\n\t}"
        : "=l"(r)
        : "f"(a), "l"(b), "l"(acc));
    return r;
}
// acc = fmaf(a_i, b_i, acc) for two pairs (cosine on normalised rows, D6)
__device__ __forceinline__ unsigned long long f2_ip(float a, unsigned long long b, unsigned long long acc) {
    unsigned long long r;
    asm("{\n\t.reg .b64 aa;\n\tmov.b64 aa, {%1, %1};\n\tfma.rn.f32x2 %0, aa, %2, %3;\n\t}"
        : "=l"(r)
        : "f"(a), "l"(b), "l"(acc));
    return r;
}
__device__ __forceinline__ float f2_lo(unsigned long long v) { return __uint_as_float(static_cast<uint32_t>(v)); }
__device__ __forceinline__ float f2_hi(unsigned long long v) { return __uint_as_float(static_cast<uint32_t>(v >> 32)); }

__device__ __forceinline__ void named_bar(int id, int threads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
// TMA row gather: 4 rows (ids r0..r3) of a 2-D tensor map (box: one 128-B
// row slab starting at element column col) land as 4 consecutive 128-B rows
// at dst (SW128 swizzle applied by the TMA unit); completion counted in
// bytes on bar
__device__ __forceinline__ void tma_gather4(void* dst, const CUtensorMap* tm, int r0, int r1, int r2, int r3,
                                            uint64_t* bar, int col = 0) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
        "%4, %5, %6}], [%7];" ::"r"(smem_u32(dst)),
        "l"(tm), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(smem_u32(bar))
        : "memory");
}



template <typename T, int MET, int STAGES, bool PK = false>
struct WsCfg {
    using E = typename std::conditional<MET == kMetCos, float, T>::type;
    static constexpr int SD = SlabCfg<T>::kDims;
    // PK (float rows): the pair-interleaved stage of the packed FP32x2 tile.
    // Slots 2j and 2j+1 share one 256-B "pair row" whose 16-B chunk c holds
    // {s0[2c], s1[2c], s0[2c+1], s1[2c+1]} of the 32-dim slab, so one
    // LDS.128 yields two packed column pairs {b0_i, b1_i} (FADD2/FFMA2
    // operands) or four row scalars.  Chunk c sits at position
    // ((c & 1) << 3) | (c >> 1) (even chunks in the first 128 B: the
    // gather's 8-lane phases write distinct bank groups), and 4-slot groups
    // are 528 B apart (16-B pad), so blocks of different 4-row groups read
    // different bank groups without any address swizzle.
    static constexpr bool kPair = PK && std::is_same<E, float>::value;
    static constexpr int kGroupFloats = 132;  // 2 pair rows of 64 floats + 4 pad
    // otherwise: 128-B row slabs (32 f32 or 128 u8 dims) whose 16-B chunks
    // are XOR-swizzled by (slot >> 2) & 7, so the LDS.128 of lanes on
    // different 4-row groups never share a bank group (padding cannot: rows
    // 4 apart always collide).
    static constexpr bool kSwz = true;
    static constexpr int RS = SD;
    static_assert(SD * sizeof(E) == 128, "row slabs are 128 B");
    static constexpr size_t kStageBytes =
        kPair ? sizeof(float) * kGroupFloats * (kWsSlots / 4) : sizeof(E) * kWsSlots * RS;
    static constexpr size_t kMetaOff = kStageBytes * STAGES;
    static constexpr size_t kPartOff = (kMetaOff + sizeof(WsMeta) * kWsMeta + 15) & ~size_t(15);
    static constexpr size_t kPartBytes = sizeof(unsigned long long) * 8 * kWsBlocks;  // row + col minima
    static constexpr size_t kEpiOff = kPartOff + 2 * kPartBytes;  // epilogue key/target staging
    static constexpr size_t kBarOff = kEpiOff + (8 + 4) * kEpiRounds * kWsEpiThreads * kWsEpiGroups;
    static constexpr int kNumBars = 2 * STAGES + 2 * kWsMeta + 4;
    // lead's double-buffered chunk cache: (m, q) bytes of 32 nodes, then
    // their Gn and Go sample-id rows (cap <= 2 * p_max = 32 ids each)
    static constexpr size_t kCacheOff = (kBarOff + 8 * kNumBars + 15) & ~size_t(15);
    static constexpr size_t kCacheBytes = 2 * 64 + 2 * 32 * 2 * 32 * sizeof(uint32_t);
    static constexpr size_t kSmem = kCacheOff + kCacheBytes;
    static_assert(kSmem + 1024 <= 232448, "227 KB dynamic shared memory per CTA (+ 1 KB TMA alignment)");
};

#ifdef KNNG_WS_PROF
// profiling build only (make WSPROF=1; tools/join_probe.py): role probes
// (1 consumers skip the math, 2 gathers skip the loads, 4 no filing) and
// cycles spent per wait site (probe bit 32)
__device__ int g_ws_probe;
__device__ unsigned long long g_ws_prof[32];
#define WS_PROBE() (*(volatile int*)&g_ws_probe)
#define WS_T0(v) const long long v = clock64()
#define WS_ACC(v, site)                                                                         \
    do {                                                                                        \
        if ((probe & 32) && (threadIdx.x & 31) == 0)                                            \
            atomicAdd(&g_ws_prof[site], static_cast<unsigned long long>(clock64() - (v)));      \
    } while (0)
#else
#define WS_PROBE() 0
#define WS_T0(v)
#define WS_ACC(v, site)
#endif

template <bool SUSP>
__device__ __forceinline__ void ws_idle_wait(uint64_t* bar, uint32_t parity, int site = 31, int probe = 0) {
#ifdef KNNG_WS_PROF
    const long long t0 = clock64();
#endif
    if constexpr (SUSP) mbar_wait_idle(bar, parity);
    else mbar_wait_sleep(bar, parity);
#ifdef KNNG_WS_PROF
    if ((probe & 32) && (threadIdx.x & 31) == 0)
        atomicAdd(&g_ws_prof[site], static_cast<unsigned long long>(clock64() - t0));
#endif
}

template <typename T, int MET, int STAGES, bool PK = false>
__global__ void __launch_bounds__(kWsThreads, 1)
k_join_ws(const T* __restrict__ X, const float* __restrict__ Xn, Dims D, Graph G, Samples S, int64_t boundary,
          unsigned long long* __restrict__ work, DevStats* __restrict__ stats) {
    using Cfg = WsCfg<T, MET, STAGES, PK>;
    using E = typename Cfg::E;
    constexpr bool kFloat = std::is_same<E, float>::value;
    using Acc = typename std::conditional<kFloat, float, unsigned int>::type;
    constexpr int SD = Cfg::SD, RS = Cfg::RS;
    const E* __restrict__ V = MET == kMetCos ? reinterpret_cast<const E*>(Xn) : reinterpret_cast<const E*>(X);

    extern __shared__ __align__(128) unsigned char ws_raw[];
    unsigned char* ws_smem = ws_raw;
    E* ring = reinterpret_cast<E*>(ws_smem);
    WsMeta* meta = reinterpret_cast<WsMeta*>(ws_smem + Cfg::kMetaOff);
    unsigned long long* parts = reinterpret_cast<unsigned long long*>(ws_smem + Cfg::kPartOff);  // [2][8][blocks]
    unsigned long long* ep_key = reinterpret_cast<unsigned long long*>(ws_smem + Cfg::kEpiOff);
    uint32_t* ep_tgt = reinterpret_cast<uint32_t*>(ep_key + kEpiRounds * kWsEpiThreads * kWsEpiGroups);
    uint64_t* bars = reinterpret_cast<uint64_t*>(ws_smem + Cfg::kBarOff);
    uint64_t* full = bars;                          // [STAGES]  producers -> consumers
    uint64_t* empty = bars + STAGES;                // [STAGES]  consumers -> producers
    uint64_t* mfull = bars + 2 * STAGES;            // [kWsMeta] lead -> all
    uint64_t* mempty = mfull + kWsMeta;             // [kWsMeta] epilogue -> lead
    uint64_t* pfull = mempty + kWsMeta;             // [2]       consumers -> epilogue
    uint64_t* pempty = pfull + 2;                   // [2]       epilogue -> consumers

    const int tid = threadIdx.x;
    const int warp = tid >> 5;
    const uint32_t lane = lane_id();
    const int d = D.d, cap = D.cap;
    const int nslab = (d + SD - 1) / SD;
    const bool restricted = boundary >= 0;
    const int probe = WS_PROBE();

    if (tid == 0) {
        for (int s = 0; s < STAGES; ++s) {
            // non-packed: one cp.async arrive per gather thread; packed: one
            // arrive per gather warp (each arrive wakes the CTA's suspended
            // waiters: 224 per slab made the idle roles spin)
            mbar_init(full + s, Cfg::kPair ? kWsGatherWarps : kWsProdThreads);
            mbar_init(empty + s, kWsConsumerWarps);
        }
        for (int s = 0; s < kWsMeta; ++s) {
            mbar_init(mfull + s, 32);
            mbar_init(mempty + s, 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(pfull + s, kWsConsumerWarps);
            mbar_init(pempty + s, 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    // warp roles: [0, 8) consumers, [8, 11) gather, 11 lead, [12, 16) epilogue.
    // The issue arbiter serves the highest warp id first: the light roles
    // (which sleep when idle) get priority so they never starve the
    // pipeline; the consumers take every remaining slot.
    if (warp >= kWsConsumerWarps + kWsProducerWarps) {
        // ================================ epilogue ===============================
        // kWsEpiGroups groups take alternate batches, so the filing latency
        // of one batch overlaps the next one's
        const int g = (warp - kWsConsumerWarps - kWsProducerWarps) / kWsEpiGroupWarps;
        const int et = tid - (kWsConsumerWarps + kWsProducerWarps) * 32 - g * kWsEpiThreads;
        unsigned long long* gkey = ep_key + g * kEpiRounds * kWsEpiThreads;
        uint32_t* gtgt = ep_tgt + g * kEpiRounds * kWsEpiThreads;
        unsigned long long n_cand = 0, n_app = 0;
        for (uint32_t b = g;; b += kWsEpiGroups) {
            const int mb = b % kWsMeta, pb = b & 1;
            ws_idle_wait<Cfg::kPair>(mfull + mb, (b / kWsMeta) & 1, 0, probe);
            const WsMeta& M = meta[mb];
            const int nn = M.nnodes;
            if (nn == 0) break;
            ws_idle_wait<Cfg::kPair>(pfull + pb, (b >> 1) & 1, 1, probe);
            WS_T0(t_sel);
            const unsigned long long* rowp = parts + pb * 8 * kWsBlocks;
            const unsigned long long* colp = rowp + 4 * kWsBlocks;
            // output o of the batch is key j of node i (obase[i] <= o): c_nn(u_j)
            // (j < m), c_no(u_{j-m}) (j < 2m), c_on(w_{j-2m})
            const int total = M.obase[nn];
            for (int r = 0; r < kEpiRounds; ++r) {
                const int o = et + r * kWsEpiThreads;
                uint64_t v = kSentinel;
                uint32_t tgt = 0;
                if (o < total) {
                    int i = 0;  // the last node with obase[i] <= o
#pragma unroll
                    for (int step = 16; step > 0; step >>= 1)
                        if (i + step < nn && M.obase[i + step] <= o) i += step;
                    const int j = o - M.obase[i];
                    const int mi = M.m[i], qi = M.q[i];
                    const int mgi = (mi + 3) >> 2, qgi = (qi + 3) >> 2, bb = M.bbase[i];
                    const int nnn_i = mgi * (mgi + 1) / 2;
                    if (j < 2 * mi) {
                        const int u = j < mi ? j : j - mi, I = u >> 2, rr = u & 3;
                        if (j < mi) {  // as a row of blocks (I, J <= I) and a column of (I' >= I, I)
                            for (int J = 0; J <= I; ++J) {
                                const uint64_t t = rowp[(bb + I * (I + 1) / 2 + J) * 4 + rr];
                                v = t < v ? t : v;
                            }
                            for (int I2 = I; I2 < mgi; ++I2) {
                                const uint64_t t = colp[(bb + I2 * (I2 + 1) / 2 + I) * 4 + rr];
                                v = t < v ? t : v;
                            }
                        } else {  // rows of the NEW-OLD blocks (I, J)
                            for (int J = 0; J < qgi; ++J) {
                                const uint64_t t = rowp[(bb + nnn_i + I * qgi + J) * 4 + rr];
                                v = t < v ? t : v;
                            }
                        }
                    } else {  // columns of the NEW-OLD blocks (I, J_w)
                        const int oo = j - 2 * mi, J = oo >> 2, c = oo & 3;
                        for (int I = 0; I < mgi; ++I) {
                            const uint64_t t = colp[(bb + nnn_i + I * qgi + J) * 4 + c];
                            v = t < v ? t : v;
                        }
                    }
                    // target: the NEW sample u_j (c_nn, c_no) or the OLD sample w_j (c_on)
                    const int sbi = M.sbase[i], mpi = (mi + 3) & ~3;
                    tgt = M.ids[j < mi ? sbi + j : (j < 2 * mi ? sbi + j - mi : sbi + mpi + j - 2 * mi)];
                }
                gkey[r * kWsEpiThreads + et] = v;
                gtgt[r * kWsEpiThreads + et] = tgt;
            }
            // partials and metadata are no longer needed: release them so the
            // consumers and the lead producer run ahead of the filing
            WS_ACC(t_sel, 12);
            named_bar(2 + g, kWsEpiThreads);
            if (et == 0) {
                mbar_arrive(pempty + pb);
                mbar_arrive(mempty + mb);
            }
            WS_T0(t_file);
            // file the keys into their targets' buckets (the k_cand_scatter
            // step, fused); keys >= the target's iteration-start k-th key
            // cannot enter (exact, D17).  All loads, then all atomics, then
            // all stores: kEpiRounds independent chains in flight per thread.
            uint64_t kv[kEpiRounds], th[kEpiRounds], bo[kEpiRounds];
            uint32_t tg[kEpiRounds], sl[kEpiRounds];
#pragma unroll
            for (int r = 0; r < kEpiRounds; ++r) {
                kv[r] = gkey[r * kWsEpiThreads + et];
                tg[r] = gtgt[r * kWsEpiThreads + et];
                th[r] = 0;
                bo[r] = 0;
                if (kv[r] != kSentinel) {  // D15: (inf, inf) inserts nothing
                    th[r] = __ldg(G.kth_t + tg[r]);
                    if (!G.rec_cnt) bo[r] = __ldg(G.boff + tg[r]);
                }
            }
            if (G.rec_cnt) {
                // record mode (distributed refine): (target, key) records,
                // one slot atomic per warp and round (warp-uniform loop)
#pragma unroll
                for (int r = 0; r < kEpiRounds; ++r) {
                    n_cand += kv[r] != kSentinel;
                    const bool ok = kv[r] != kSentinel && kv[r] < th[r];
                    n_app += ok;
                    const uint32_t b = __ballot_sync(kFull, ok);
                    unsigned long long wb = 0;
                    if (lane == 0 && b) wb = atomicAdd(G.rec_cnt, static_cast<unsigned long long>(__popc(b)));
                    const uint64_t slot = shfl_u64(wb, 0) + __popc(b & lanemask_lt());
                    if (ok) {
                        G.rec_key[slot] = kv[r];
                        G.rec_tgt[slot] = tg[r];
                    }
                }
                continue;
            }
            if (probe & 4) continue;
#pragma unroll
            for (int r = 0; r < kEpiRounds; ++r) {
                n_cand += kv[r] != kSentinel;
                const bool ok = kv[r] != kSentinel && kv[r] < th[r];
                n_app += ok;
                sl[r] = ok ? atomicAdd(G.bcnt + tg[r], 1u) : 0xFFFFFFFFu;
            }
#pragma unroll
            for (int r = 0; r < kEpiRounds; ++r)
                if (sl[r] != 0xFFFFFFFFu) G.bucket[bo[r] + sl[r]] = kv[r];
            WS_ACC(t_file, 13);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            n_cand += __shfl_xor_sync(kFull, n_cand, o);
            n_app += __shfl_xor_sync(kFull, n_app, o);
        }
        if (lane == 0) {
            if (n_cand) atomicAdd(&stats->candidates, n_cand);
            if (n_app) atomicAdd(&stats->appended, n_app);
        }
        return;
    }

    if (warp >= kWsConsumerWarps) {
        // =============================== producers ==============================
        const int ptid = tid - kWsConsumerWarps * 32;  // gather thread index
        constexpr int CE = SlabCfg<T>::kChunkElems, CPR = SD / CE;
        uint32_t slab_it = 0, meta_it = 0;
        // each gather thread owns one 16-B chunk column of the slab and walks
        // the rows: one shared id load, one address, one copy per chunk
        static_assert(kWsProdThreads % CPR == 0, "gather threads must tile the chunk columns");
        constexpr int kRowsPerPass = kWsProdThreads / CPR;
        const int part = ptid % CPR;
        const int row0 = ptid / CPR;
        // packed layout: each task is (pair row j, 16-B column c4 of the
        // slab): two LDG.128 (slots 2j, 2j+1, dims 4c4..4c4+3), interleaved
        // in registers into chunks 2c4 and 2c4+1 (two STS.128).  All of a
        // slab's loads are issued before the stage is awaited, then stored,
        // then the stage's full barrier is arrived on (release: the stores
        // are visible to the consumers that observe the phase).
        constexpr int kTaskPerThr = (kWsSlots / 2 * 8 + kWsProdThreads - 1) / kWsProdThreads;
        auto gather_pk = [&](const WsMeta& M) {
            const int npairs = M.nslots >> 1;
            for (int sl = 0; sl < nslab; ++sl) {
                const int st = slab_it % STAGES;
                const int ncol = min(SD, d - sl * SD) >> 2;  // 16-B columns in this slab (d % 4 == 0)
                float4 r0[kTaskPerThr], r1[kTaskPerThr];
#pragma unroll
                for (int i = 0; i < kTaskPerThr; ++i) {
                    const int task = ptid + i * kWsProdThreads, j = task >> 3, c4 = task & 7;
                    r0[i] = make_float4(0.f, 0.f, 0.f, 0.f);
                    r1[i] = r0[i];
                    if (j < npairs && c4 < ncol && !(probe & 2)) {
                        const uint32_t i0 = M.ids[2 * j], i1 = M.ids[2 * j + 1];
                        const E* src = V + sl * SD + 4 * c4;
                        if (i0 != 0xFFFFFFFFu) r0[i] = __ldg(reinterpret_cast<const float4*>(src + static_cast<size_t>(i0) * d));
                        if (i1 != 0xFFFFFFFFu) r1[i] = __ldg(reinterpret_cast<const float4*>(src + static_cast<size_t>(i1) * d));
                    }
                }
                ws_idle_wait<Cfg::kPair>(empty + st, ((slab_it / STAGES) & 1) ^ 1, 2, probe);
                float* stage = reinterpret_cast<float*>(ring) + static_cast<size_t>(st) * (Cfg::kStageBytes / 4);
#pragma unroll
                for (int i = 0; i < kTaskPerThr; ++i) {
                    const int task = ptid + i * kWsProdThreads, j = task >> 3, c4 = task & 7;
                    if (j < npairs && c4 < ncol) {
                        float* row = stage + (j >> 1) * Cfg::kGroupFloats + (j & 1) * 64;
                        *reinterpret_cast<float4*>(row + 4 * c4) = make_float4(r0[i].x, r1[i].x, r0[i].y, r1[i].y);
                        *reinterpret_cast<float4*>(row + 32 + 4 * c4) = make_float4(r0[i].z, r1[i].z, r0[i].w, r1[i].w);
                    }
                }
                __syncwarp();  // the warp's stores before its one release arrive
                if (lane == 0) mbar_arrive(full + st);
                ++slab_it;
            }
        };
        auto gather = [&](const WsMeta& M) {
            if constexpr (Cfg::kPair) {
                gather_pk(M);
                return;
            }
            const int nslots = M.nslots;
            for (int sl = 0; sl < nslab; ++sl) {
                const int st = slab_it % STAGES;
                ws_idle_wait<Cfg::kPair>(empty + st, ((slab_it / STAGES) & 1) ^ 1, 3, probe);
                const int e0 = sl * SD + part * CE;
                E* dst = ring + static_cast<size_t>(st) * kWsSlots * RS;
                const E* src0 = V + e0;
                if (sl * SD + SD <= d) {  // full slab: plain 16-B copies
                    for (int slot = row0; slot < nslots; slot += kRowsPerPass) {
                        const uint32_t id = M.ids[slot];
                        if (id == 0xFFFFFFFFu) continue;
                        const int c = Cfg::kSwz ? (part ^ ((slot >> 2) & 7)) : part;
                        const uint32_t s = smem_u32(dst + slot * RS + c * CE);
                        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s),
                                     "l"(src0 + static_cast<size_t>(id) * d));
                    }
                } else if (e0 < d) {  // last partial slab: zero-filled copies
                    const int bytes = min(CE, d - e0) * static_cast<int>(sizeof(E));
                    for (int slot = row0; slot < nslots; slot += kRowsPerPass) {
                        const uint32_t id = M.ids[slot];
                        if (id == 0xFFFFFFFFu) continue;
                        const int c = Cfg::kSwz ? (part ^ ((slot >> 2) & 7)) : part;
                        cp_async16(dst + slot * RS + c * CE, src0 + static_cast<size_t>(id) * d, bytes);
                    }
                }
                asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(full + st))
                             : "memory");
                ++slab_it;
            }
        };
        if (warp < kWsConsumerWarps + kWsGatherWarps) {  // gather warps follow the batch stream
            while (true) {
                const int mb = meta_it % kWsMeta;
                ws_idle_wait<Cfg::kPair>(mfull + mb, (meta_it / kWsMeta) & 1, 4, probe);
                const WsMeta& M = meta[mb];
                if (M.nnodes == 0) break;
                gather(M);
                ++meta_it;
            }
            return;
        }
        // lead producer: forms batches and publishes their metadata, running
        // up to kWsMeta batches ahead of the gathers and the tiles.  Chunks
        // of 32 nodes are claimed two ahead, and the next chunk's counts and
        // sample-id rows are prefetched with cp.async into a double-buffered
        // chunk cache while the current chunk's batches are published, so
        // publication never waits on global memory.
        uint8_t* cc_cnt = ws_smem + Cfg::kCacheOff;                                      // [2][64]
        uint32_t* cc_ids = reinterpret_cast<uint32_t*>(ws_smem + Cfg::kCacheOff + 128);  // [2][32][2cap]
        int cur_buf = 0;
        int64_t cur_x0 = 0;
        auto claim = [&]() -> unsigned long long {
            unsigned long long c0 = 0;
            if (lane == 0) c0 = atomicAdd(work, 32ull);
            return c0;  // lane 0's value; broadcast at use
        };
        auto fetch = [&](int buf, int64_t xb) {
            if (xb < D.n) {
                const int nodes = static_cast<int>(D.n - xb < 32 ? D.n - xb : 32);
                uint8_t* ccnt = cc_cnt + buf * 64;
                uint32_t* cids = cc_ids + static_cast<size_t>(buf) * 32 * 2 * cap;
                if (lane < 16) {  // (m, q) byte pairs, 4 bytes per lane, zero-filled past n
                    const int lo = 4 * lane, bytes = max(0, min(4, 2 * nodes - lo));
                    const uint32_t s = smem_u32(ccnt + lo);
                    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(s),
                                 "l"(S.gcnt + 2 * xb + lo), "r"(bytes)
                                 : "memory");
                }
                if ((cap & 3) == 0) {
                    // 16-B copies, node-major: lane -> (node of the pass, chunk of its Gn|Go rows)
                    const int cpr = cap >> 2, per_node = 2 * cpr, npi = 32 / per_node;
                    const int sub = static_cast<int>(lane) / per_node, c = static_cast<int>(lane) - sub * per_node;
                    const uint32_t* base = (c < cpr ? S.G : S.G + static_cast<size_t>(D.n) * cap) + 4 * (c < cpr ? c : c - cpr);
                    for (int nb = 0; nb < nodes; nb += npi) {
                        const int node = nb + sub;
                        if (sub < npi && node < nodes) {
                            const uint32_t s = smem_u32(cids + node * 2 * cap + 4 * c);
                            asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(s),
                                         "l"(base + static_cast<size_t>(xb + node) * cap)
                                         : "memory");
                        }
                    }
                } else {
                    for (int node = 0; node < nodes; ++node)
                        for (int w = lane; w < 2 * cap; w += 32) {
                            const uint32_t* src = w < cap ? S.G + static_cast<size_t>(xb + node) * cap + w
                                                          : S.G + static_cast<size_t>(D.n) * cap +
                                                                static_cast<size_t>(xb + node) * cap + (w - cap);
                            const uint32_t s = smem_u32(cids + node * 2 * cap + w);
                            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(src) : "memory");
                        }
                }
            }
            cp_async_commit();
        };
        int64_t x0 = static_cast<int64_t>(__shfl_sync(kFull, claim(), 0));
        int64_t xnext = static_cast<int64_t>(__shfl_sync(kFull, claim(), 0));
        int buf = 0;
        fetch(0, x0);
        int cur = 32;  // position inside the current 32-node chunk
        int my_m = 0, my_q = 0, my_nb = 0, my_sl = 0;
        int p_nb = 0, p_sl = 0, p_co = 0;  // chunk prefix sums of blocks, slots, selected keys
        unsigned long long n_joins = 0, n_m = 0, n_q = 0, n_rows = 0;
        while (true) {
            if (cur >= 32) {
                if (x0 >= D.n) break;
                WS_T0(t_chunk);
                const unsigned long long claimed = claim();  // used one chunk later
                fetch(buf ^ 1, xnext);
                cp_async_wait<1>();  // this chunk's group has landed
                __syncwarp();  // every lane's copies of this chunk visible to all
                const int64_t x = x0 + lane;
                my_m = 0;
                my_q = 0;
                if (x < D.n) {
                    my_m = cc_cnt[buf * 64 + 2 * lane];
                    my_q = cc_cnt[buf * 64 + 2 * lane + 1];
                }
                if (my_m == 0) my_q = 0;  // no NEW sample: nothing to join
                if (my_m > 0) {  // the join counters keep the method's m and q
                    ++n_joins;
                    n_m += my_m;
                    n_q += my_q;
                }
                if (restricted && my_m > 0) {
                    // GGM refine (D22): NEW samples are all cross-subset, so
                    // only (NEW, own-subset OLD) pairs remain; keep the
                    // own-subset OLD ids in place (id order kept), skip a node
                    // without any.  Same candidates and counts, fewer rows.
                    uint32_t* orow = cc_ids + static_cast<size_t>(buf) * 32 * 2 * cap + lane * 2 * cap + cap;
                    const bool xs = D.base + x >= boundary;
                    int qq = 0;
                    for (int j = 0; j < my_q; ++j) {
                        const uint32_t id = orow[j];
                        if ((static_cast<int64_t>(id) >= boundary) == xs) orow[qq++] = id;
                    }
                    my_q = qq;
                    if (qq == 0) my_m = 0;
                }
                const int mg = (my_m + 3) >> 2, qg = (my_q + 3) >> 2;
                my_nb = mg * (mg + 1) / 2 + mg * qg;
                my_sl = 4 * (mg + qg);
                // inclusive prefix sums over the chunk's 32 nodes, once per
                // chunk: a batch's bounds are then differences (no per-batch
                // shuffle scans -- the lead's shuffles queue behind the
                // consumers' shared-memory traffic)
                p_nb = my_nb;
                p_sl = my_sl;
                p_co = 2 * my_m + my_q;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int tb = __shfl_up_sync(kFull, p_nb, o), ts = __shfl_up_sync(kFull, p_sl, o);
                    const int tc = __shfl_up_sync(kFull, p_co, o);
                    if (static_cast<int>(lane) >= o) {
                        p_nb += tb;
                        p_sl += ts;
                        p_co += tc;
                    }
                }
                cur = 0;
                cur_buf = buf;
                cur_x0 = x0;
                x0 = xnext;
                xnext = static_cast<int64_t>(__shfl_sync(kFull, claimed, 0));
                buf ^= 1;
                WS_ACC(t_chunk, 11);
            }
            // take nodes cur.. while the batch's blocks and slots fit
            // bounds relative to the chunk prefix before node `cur`
            const int src0 = cur > 0 ? cur - 1 : 0;
            int b_nb = __shfl_sync(kFull, p_nb, src0), b_sl = __shfl_sync(kFull, p_sl, src0);
            int b_co = __shfl_sync(kFull, p_co, src0);
            if (cur == 0) b_nb = b_sl = b_co = 0;
            const bool pending = static_cast<int>(lane) >= cur;
            const bool fits = pending && p_nb - b_nb <= kWsBlocks && p_sl - b_sl <= kWsSlots;
            const uint32_t fm = __ballot_sync(kFull, fits);
            const int end = fm ? 32 - __clz(fm) : cur;  // fits is a prefix of [cur, 32)
            const int src1 = end - 1 < 0 ? 0 : end - 1;
            const int nb_tot = __shfl_sync(kFull, p_nb, src1) - b_nb;
            const int ns_tot = __shfl_sync(kFull, p_sl, src1) - b_sl;
            const int no_tot = __shfl_sync(kFull, p_co, src1) - b_co;
            const int first = cur;
            cur = end;
            if (end <= first || nb_tot == 0) continue;  // only nodes without NEW samples
            // ---- publish batch metadata: every lane its own node (no
            // per-node shuffles)
            const int mb = meta_it % kWsMeta;
            ws_idle_wait<Cfg::kPair>(mempty + mb, ((meta_it / kWsMeta) & 1) ^ 1, 5, probe);
            WsMeta& M = meta[mb];
            WS_T0(t_pub);
            const int nn = end - first;
            const bool in_batch = static_cast<int>(lane) >= first && static_cast<int>(lane) < end;
            if (in_batch) {
                const int i = lane - first;
                const int sb = p_sl - my_sl - b_sl;
                M.x[i] = cur_x0 + lane;
                M.m[i] = my_m;
                M.q[i] = my_q;
                M.sbase[i] = sb;
                M.bbase[i] = p_nb - my_nb - b_nb;
                M.obase[i] = p_co - (2 * my_m + my_q) - b_co;
                n_rows += my_m + my_q;
                // the sample ids of my slots, from the chunk cache
                const uint32_t* row = cc_ids + static_cast<size_t>(cur_buf) * 32 * 2 * cap + lane * 2 * cap;
                const int mpad = (my_m + 3) & ~3;
                for (int js = 0; js < my_sl; ++js) {
                    uint32_t id = 0xFFFFFFFFu;
                    if (js < my_m) id = row[js];
                    else if (js >= mpad && js - mpad < my_q) id = row[cap + (js - mpad)];
                    M.ids[sb + js] = id;
                }
            }
            if (lane == 0) {
                M.nnodes = nn;
                M.nblocks = nb_tot;
                M.nslots = ns_tot;
                M.bbase[nn] = nb_tot;
                M.obase[nn] = no_tot;
            }
            __syncwarp();
            WS_ACC(t_pub, 10);
            mbar_arrive(mfull + mb);  // all 32 lanes: releases every lane's writes
            ++meta_it;
        }
        cp_async_wait<0>();  // no prefetch outstanding at exit
        // termination markers: one per epilogue group (each group waits on
        // its own batch sequence); consumers and gatherers stop at the first
        for (int e = 0; e < kWsEpiGroups; ++e) {
            const int mb = meta_it % kWsMeta;
            ws_idle_wait<Cfg::kPair>(mempty + mb, ((meta_it / kWsMeta) & 1) ^ 1, 6, probe);
            if (lane == 0) meta[mb].nnodes = 0;
            __syncwarp();
            mbar_arrive(mfull + mb);
            ++meta_it;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            n_joins += __shfl_xor_sync(kFull, n_joins, o);
            n_m += __shfl_xor_sync(kFull, n_m, o);
            n_q += __shfl_xor_sync(kFull, n_q, o);
            n_rows += __shfl_xor_sync(kFull, n_rows, o);
        }
        if (lane == 0 && n_joins) {
            atomicAdd(&stats->joins, n_joins);
            atomicAdd(&stats->sum_m, n_m);
            atomicAdd(&stats->sum_q, n_q);
            atomicAdd(&stats->rows, n_rows);
        }
        return;
    }

    // ================================ consumers =================================
    const int ct = tid;  // 0 .. kWsBlocks-1
    uint32_t slab_it = 0;
    unsigned long long my_pairs = 0;
    for (uint32_t b = 0;; ++b) {
        const int mb = b % kWsMeta, pb = b & 1;
        if constexpr (Cfg::kPair) mbar_wait(mfull + mb, (b / kWsMeta) & 1);  // the critical role spins
        else ws_idle_wait<false>(mfull + mb, (b / kWsMeta) & 1, 7, probe);
        const WsMeta& M = meta[mb];
        const int nn = M.nnodes;
        if (nn == 0) break;
        // ---- my block
        const bool active = ct < M.nblocks;
        // my block's node: the last i with bbase[i] <= ct (binary search)
        int nd = 0;
        if (active) {
#pragma unroll
            for (int step = 16; step > 0; step >>= 1)
                if (nd + step < nn && M.bbase[nd + step] <= ct) nd += step;
        }
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
        constexpr int RW = RS;  // ring distance between a block's rows
        const int fA = ((sb + rb) >> 2) & 7, fB = ((sb + cb) >> 2) & 7;  // chunk swizzle

        Acc acc[4][4];
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
            for (int c = 0; c < 4; ++c) acc[r][c] = Acc(0);
        // packed accumulators: acc2[r][h] = {acc[r][2h], acc[r][2h+1]}
        unsigned long long acc2[4][2];
#pragma unroll
        for (int r = 0; r < 4; ++r) acc2[r][0] = acc2[r][1] = 0ull;

        for (int sl = 0; sl < nslab; ++sl) {
            const int st = slab_it % STAGES;
            mbar_wait(full + st, (slab_it / STAGES) & 1);
            WS_T0(t_slab);
            if constexpr (Cfg::kPair) {
                if (active && !(probe & 1)) {
                    // rows rb..rb+3 and columns cb..cb+3 are 4-slot groups
                    const float* stage = reinterpret_cast<const float*>(ring) + static_cast<size_t>(st) * (Cfg::kStageBytes / 4);
                    const float* A = stage + ((sb + rb) >> 2) * Cfg::kGroupFloats;
                    const float* B = stage + ((sb + cb) >> 2) * Cfg::kGroupFloats;
                    const int nc = min(SD, d - sl * SD) >> 1;  // 2-dim chunks, in dimension order
#pragma unroll
                    for (int c = 0; c < SD / 2; ++c) {
                        if (c >= nc) break;
                        const int pos = (((c & 1) << 3) | (c >> 1)) * 4;
                        const float4 a01 = *reinterpret_cast<const float4*>(A + pos);       // r0,r1 @2c; r0,r1 @2c+1
                        const float4 a23 = *reinterpret_cast<const float4*>(A + 64 + pos);  // r2,r3
                        const ulonglong2 b01 = *reinterpret_cast<const ulonglong2*>(B + pos);       // {c0,c1} @2c, @2c+1
                        const ulonglong2 b23 = *reinterpret_cast<const ulonglong2*>(B + 64 + pos);  // {c2,c3}
                        const float ar[2][4] = {{a01.x, a01.y, a23.x, a23.y}, {a01.z, a01.w, a23.z, a23.w}};
                        const unsigned long long bp[2][2] = {{b01.x, b23.x}, {b01.y, b23.y}};
#pragma unroll
                        for (int h = 0; h < 2; ++h)
#pragma unroll
                            for (int r = 0; r < 4; ++r)
#pragma unroll
                                for (int cp = 0; cp < 2; ++cp) {
                                    if constexpr (MET == kMetCos) {
                                        acc2[r][cp] = f2_ip(ar[h][r], bp[h][cp], acc2[r][cp]);
                                    } else if constexpr (MET == kMetChi2) {
                                        float lo = f2_lo(acc2[r][cp]), hi = f2_hi(acc2[r][cp]);
                                        lo = chi2_term(ar[h][r], f2_lo(bp[h][cp]), lo);
                                        hi = chi2_term(ar[h][r], f2_hi(bp[h][cp]), hi);
                                        acc2[r][cp] = (static_cast<unsigned long long>(__float_as_uint(hi)) << 32) |
                                                      __float_as_uint(lo);
                                    } else {
                                        acc2[r][cp] = f2_l2(ar[h][r], bp[h][cp], acc2[r][cp]);
                                    }
                                }
                    }
                }
            } else if (active) {
                const E* __restrict__ A = ring + static_cast<size_t>(st) * kWsSlots * RS + aoff;
                const E* __restrict__ B = ring + static_cast<size_t>(st) * kWsSlots * RS + boff;
                const int lim = min(SD, d - sl * SD);
                if constexpr (kFloat) {
#pragma unroll 2
                    for (int i = 0; i < SD; i += 4) {
                        if (i >= lim) break;
                        float4 a[4], bv[4];
#pragma unroll
                        for (int r = 0; r < 4; ++r)
                            a[r] = *reinterpret_cast<const float4*>(A + r * RW + (((i >> 2) ^ fA) << 2));
#pragma unroll
                        for (int c = 0; c < 4; ++c)
                            bv[c] = *reinterpret_cast<const float4*>(B + c * RW + (((i >> 2) ^ fB) << 2));
#pragma unroll
                        for (int r = 0; r < 4; ++r)
#pragma unroll
                            for (int c = 0; c < 4; ++c) {
                                if constexpr (MET == kMetCos) {
                                    acc[r][c] = fmaf(a[r].x, bv[c].x, acc[r][c]);
                                    acc[r][c] = fmaf(a[r].y, bv[c].y, acc[r][c]);
                                    acc[r][c] = fmaf(a[r].z, bv[c].z, acc[r][c]);
                                    acc[r][c] = fmaf(a[r].w, bv[c].w, acc[r][c]);
                                } else if constexpr (MET == kMetChi2) {
                                    acc[r][c] = chi2_term(a[r].x, bv[c].x, acc[r][c]);
                                    acc[r][c] = chi2_term(a[r].y, bv[c].y, acc[r][c]);
                                    acc[r][c] = chi2_term(a[r].z, bv[c].z, acc[r][c]);
                                    acc[r][c] = chi2_term(a[r].w, bv[c].w, acc[r][c]);
                                } else {
                                    float tt;
                                    tt = a[r].x - bv[c].x; acc[r][c] = fmaf(tt, tt, acc[r][c]);
                                    tt = a[r].y - bv[c].y; acc[r][c] = fmaf(tt, tt, acc[r][c]);
                                    tt = a[r].z - bv[c].z; acc[r][c] = fmaf(tt, tt, acc[r][c]);
                                    tt = a[r].w - bv[c].w; acc[r][c] = fmaf(tt, tt, acc[r][c]);
                                }
                            }
                    }
                } else {
                    // uint8: exact integer sum of squares (D5); one LDS.128
                    // per row brings 16 dims, 2 instructions per 4 dims/pair
#pragma unroll 2
                    for (int j = 0; j < SD / 16; ++j) {
                        if (j * 16 >= lim) break;
                        uint4 a[4], bv[4];
#pragma unroll
                        for (int r = 0; r < 4; ++r) a[r] = *reinterpret_cast<const uint4*>(A + r * RW + ((j ^ fA) << 4));
#pragma unroll
                        for (int c = 0; c < 4; ++c) bv[c] = *reinterpret_cast<const uint4*>(B + c * RW + ((j ^ fB) << 4));
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
                }
            }
            WS_ACC(t_slab, 14);
            __syncwarp();
            if (lane == 0) mbar_arrive(empty + st);
            ++slab_it;
        }
        WS_T0(t_min);
        if constexpr (Cfg::kPair) {
#pragma unroll
            for (int r = 0; r < 4; ++r)
#pragma unroll
                for (int cp = 0; cp < 2; ++cp) {
                    acc[r][2 * cp] = f2_lo(acc2[r][cp]);
                    acc[r][2 * cp + 1] = f2_hi(acc2[r][cp]);
                }
        }
        // ---- block minima: 4 row keys (c_nn / c_no candidates of the NEW
        // rows) and 4 column keys (c_nn / c_on candidates of the columns)
        if constexpr (Cfg::kPair) mbar_wait(pempty + pb, ((b >> 1) & 1) ^ 1);
        else ws_idle_wait<false>(pempty + pb, ((b >> 1) & 1) ^ 1, 8, probe);
        unsigned long long* rowp = parts + pb * 8 * kWsBlocks;
        unsigned long long* colp = rowp + 4 * kWsBlocks;
        if (active) {
            const uint32_t* nid = M.ids + sb;
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
                    float dist;
                    if constexpr (MET == kMetCos) {
                        const float x1 = 1.0f - acc[r][c];
                        dist = x1 > 0.0f ? x1 : 0.0f;
                    } else if constexpr (kFloat) {
                        dist = acc[r][c];
                    } else {
                        dist = static_cast<float>(acc[r][c]);
                    }
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
        __syncwarp();
        WS_ACC(t_min, 15);
        if (lane == 0) mbar_arrive(pfull + pb);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) my_pairs += __shfl_xor_sync(kFull, my_pairs, o);
    if (lane == 0 && my_pairs) atomicAdd(&stats->dist_evals, my_pairs);
}

}  // namespace knng
