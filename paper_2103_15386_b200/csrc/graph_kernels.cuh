// graph_kernels.cuh -- init, list update + sampling, reverse sampling (CSR),
// state export.  Warp-per-node kernels: one k-NN list (k <= 32 entries) is
// one u64 key per lane, so every list operation is a register/shuffle
// operation and every list read/write is one coalesced 256-B transaction.
#pragma once
#include "common.cuh"

namespace knng {

struct DevStats {  // device mirror of knng_iter_stats
    unsigned long long joins, sum_m, sum_q, dist_evals, candidates, appended, accepted, rows, recomputed;
};

// Bucketed bulk update (D17): the candidates of one iteration for target t
// live in bucket[boff[t] .. boff[t] + bcnt[t]); boff is an exclusive scan of
// an exact upper bound of what t can receive (see k_scan_*), so a bucket can
// never overflow and no lock is needed.
struct Graph {
    uint64_t* keys;     // [n][k] ascending
    uint32_t* newmask;  // [n]    bit j = entry j is NEW
    uint64_t* kth;      // [n]    k-th key at iteration start (update threshold)
    uint32_t* bcnt;     // [n]    candidates appended to t's bucket
    const uint64_t* boff;  // [n+1] bucket offsets (= Samples::off channel 2)
    uint64_t* bucket;   // [6 n p] candidate keys of the current iteration
    // The joins read the threshold of target t at kth_t[t] (t: a sample id).
    // One GPU: kth_t == kth.  Distributed refine (dist_kernels.cuh): kth_t
    // is the group-wide copy, gathered every iteration.
    const uint64_t* kth_t;
    // Record mode (distributed refine): instead of appending into the local
    // buckets, the joins write (target, key) records at rec_tgt/rec_key[slot],
    // slot from the counter rec_cnt; nullptr = bucket mode.
    uint32_t* rec_tgt;
    uint64_t* rec_key;
    unsigned long long* rec_cnt;
    // Locked immediate update (join_locked.cuh, the ablation of P:364-366):
    // per-list (or per-segment) spinlock words and the "entered during this
    // iteration" bits, one u32 per list segment; nullptr in the bulk path.
    unsigned int* lock;
    uint32_t* imask;
};

struct Samples {
    uint32_t* fwd;   // [2][n][p]   forward NEW / OLD samples
    uint8_t* fcnt;   // [n][2]
    uint32_t* rcnt;  // [2][n]      reverse counts
    uint32_t* fpos;  // [2][n][p]   slot of forward sample (s, j) in its target's reverse list
    uint64_t* off;   // [3][n+1]    CSR offsets: reverse NEW, reverse OLD, buckets
    uint32_t* rsrc;  // [2][rstride] reverse sources
    int64_t rstride; // n*p (one GPU) or the received-record bound (distributed)
    uint32_t* G;     // [2][n][cap] G_new / G_old, sorted unique
    uint8_t* gcnt;   // [n][2]      m = |G_new|, q = |G_old|
    uint64_t* bsum;  // [3][nblk]   scan block sums
    uint64_t* cand;  // [n][3 cap]  join output: c_nn(u), c_no(u), c_on(w) keys
};

struct Dims {
    int64_t n;          // nodes whose lists this launch owns
    int d, k, p, cap;
    int64_t base = 0;   // id of the first owned node (distributed refine; else 0)
};

__device__ __forceinline__ uint32_t kmask_of(int k) { return k >= 32 ? kFull : ((1u << k) - 1u); }

// ------------------------------------------------------------------ init
// Alg. 1 lines 1-4: k distinct random ids != s (D1, D2) drawn in
// counter order j = 0, 1, ... from Philox(INIT, s, j, s >> 32), canonical
// distances, sorted by key (D3), all NEW.
// do_sample: also the first iteration's sampling step (k_merge_sample with
// no merge, fused): every entry is NEW, so FN(s) = the first min(p, k)
// entries (marked OLD, each counted in its target's reverse list), FO(s) is
// empty (D7, D12-D13).
template <typename T, int MET>
__global__ void k_init(const T* __restrict__ X, const float* __restrict__ Xn, Dims D,
                       uint64_t seed, Graph G, Samples S, int do_sample) {
    const int64_t s = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (s >= D.n) return;
    const uint32_t lane = lane_id();
    const int k = D.k;
    const uint2 key = seed_key(seed);
    extern __shared__ uint32_t init_scratch[];  // 32 u32 per warp
    uint32_t* scr = init_scratch + (threadIdx.x >> 5) * 32;
    uint32_t chosen = 0xFFFFFFFFu;
    int cnt = 0;
    for (uint32_t j0 = 0; cnt < k; j0 += 32) {
        const uint4 o = philox4x32_10(
            make_uint4(kTagInit, static_cast<uint32_t>(s), j0 + lane, static_cast<uint32_t>(static_cast<uint64_t>(s) >> 32)),
            key);
        const uint64_t r = uniform_below(o, static_cast<uint64_t>(D.n - 1));
        const uint32_t v = static_cast<uint32_t>(r + (r >= static_cast<uint64_t>(s) ? 1 : 0));
        bool dup = false;
        for (int t = 0; t < cnt; ++t) dup |= (__shfl_sync(kFull, chosen, t) == v);
        dup |= (__match_any_sync(kFull, v) & lanemask_lt()) != 0u;  // an earlier lane drew it
        const uint32_t acc = __ballot_sync(kFull, !dup);
        // accepted draw of rank r fills lane cnt + r (compaction through shared memory)
        const int slot = cnt + __popc(acc & lanemask_lt());
        __syncwarp();
        if (!dup && slot < k) scr[slot] = v;
        __syncwarp();
        const int nc = min(k, cnt + __popc(acc));
        if (static_cast<int>(lane) >= cnt && static_cast<int>(lane) < nc) chosen = scr[lane];
        cnt = nc;
    }
    uint64_t kk = kSentinel;
    if (static_cast<int>(lane) < k) {
        float dist;
        if constexpr (MET == kMetCos) {
            dist = Canon<float>::cos(Xn + static_cast<size_t>(s) * D.d, Xn + static_cast<size_t>(chosen) * D.d, D.d);
        } else if constexpr (MET == kMetChi2) {
            dist = Canon<float>::chi2(X + static_cast<size_t>(s) * D.d, X + static_cast<size_t>(chosen) * D.d, D.d);
        } else {
            dist = Canon<T>::l2(X + static_cast<size_t>(s) * D.d, X + static_cast<size_t>(chosen) * D.d, D.d);
        }
        kk = make_key(dist, chosen);
    }
    kk = warp_sort_u64(kk);
    if (static_cast<int>(lane) < k) G.keys[static_cast<size_t>(s) * k + lane] = kk;
    if (static_cast<int>(lane) == k - 1) G.kth[s] = kk;
    if (!do_sample) {
        if (lane == 0) G.newmask[s] = kmask_of(k);
        return;
    }
    const int p = D.p, fn = min(p, k);
    if (static_cast<int>(lane) < fn) {
        const uint32_t id = key_id(kk);
        S.fwd[static_cast<size_t>(s) * p + lane] = id;
        S.fpos[static_cast<size_t>(s) * p + lane] = atomicAdd(S.rcnt + id, 1u);
    }
    if (lane == 0) {
        G.newmask[s] = kmask_of(k) & ~kmask_of(fn);
        S.fcnt[2 * s] = static_cast<uint8_t>(fn);
        S.fcnt[2 * s + 1] = 0;
    }
}

// ---------------------------------------------------- list update + sample
// One warp per node s.
//  do_merge : G'[s] = k smallest unique of G[s] U bucket[s] (D16-D17);
//             survivors keep their flag, newcomers are NEW.
//  do_sample: forward samples FN(s) = first min(p, #NEW) NEW entries and
//             FO(s) = first min(p, #OLD) OLD entries in list order (P:147,
//             D7); FN entries are marked OLD (D12-D13); reverse counts
//             for the CSR of P:149.
__global__ void __launch_bounds__(256, 8) k_merge_sample(Dims D, Graph G, Samples S, int do_merge, int do_sample,
                               DevStats* __restrict__ prev_stats) {
    const int64_t s = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (s >= D.n) return;
    const uint32_t lane = lane_id();
    const int k = D.k, p = D.p;
    const bool in_list = static_cast<int>(lane) < k;
    const uint32_t mask = G.newmask[s];
    // the bucket's count and offset load with the list (one dependent
    // global round trip less before the bucket itself)
    const uint32_t bc = do_merge ? G.bcnt[s] : 0u;
    const uint64_t bo = do_merge ? G.boff[s] : 0ull;
    Elem cur{in_list ? G.keys[static_cast<size_t>(s) * k + lane] : kSentinel,
             in_list ? ((mask >> lane) & 1u) : 0u};
    bool changed = false;
    if (G.imask) {  // locked immediate update: entries that entered last iteration
        if (lane == 0) {
            const uint32_t im = G.imask[s];
            if (im && prev_stats) atomicAdd(&prev_stats->accepted, static_cast<unsigned long long>(__popc(im)));
            G.imask[s] = 0;
        }
    }
    if (do_merge) {
        const uint32_t c = bc;
        if (c > 0) {
            extern __shared__ uint64_t ms_scratch[];  // per warp: list copy, merged keys (64 u64), metas (32 u32)
            uint64_t* lst = ms_scratch + (threadIdx.x >> 5) * 80;
            uint64_t* outk = lst + 32;
            uint32_t* outm = reinterpret_cast<uint32_t*>(lst + 64);
            const uint64_t* bk = G.bucket + bo;
            for (uint32_t base = 0; base < c; base += 32) {
                const uint64_t cand = (base + lane < c) ? bk[base + lane] : kSentinel;
                // Pre-filter (exact): a candidate equal to a list key is the
                // same id (D5 keys are canonical per id) and one not below the
                // current k-th key cannot enter the k smallest.
                const uint64_t kth = shfl_u64(cur.key, k - 1);
                __syncwarp();
                lst[lane] = cur.key;
                __syncwarp();
                int pos = 0;  // list entries below cand
#pragma unroll
                for (int step = 16; step > 0; step >>= 1)
                    if (lst[pos + step - 1] < cand) pos += step;
                bool keep = cand < kth && lst[pos] != cand;
                const uint32_t km0 = __ballot_sync(kFull, keep);
                if (km0 == 0) continue;
                int* hist = reinterpret_cast<int*>(outm);  // outm / outk are free until the output step
                uint64_t* sc = outk;
                __syncwarp();
                hist[lane] = 0;
                sc[lane] = cand;
                __syncwarp();
                // candidates sharing an insertion position (one 32-bit match);
                // equal keys (the same candidate from two joins) always share
                // it: the lowest lane of each key stays
                const uint32_t grp = __match_any_sync(kFull, keep ? static_cast<uint32_t>(pos) : 64u + lane);
                const uint32_t others = keep ? (grp & ~(1u << lane)) : 0u;
                bool dup = false;
                for (uint32_t g = others & lanemask_lt(); g; g &= g - 1) dup |= sc[__ffs(g) - 1] == cand;
                const uint32_t dupm = __ballot_sync(kFull, dup);
                keep = keep && !dup;
                // Merge by ranks (no sorting network): a survivor lands at
                // (list entries below it) + (survivors below it); a list entry
                // moves down by the survivors below it; past slot k: dropped.
                // No per-survivor loop: the list separates the survivors, so
                // survivor x is below list entry i iff pos(x) <= i -- the
                // shifts are the prefix counts of a histogram of the
                // insertion positions, and a survivor's rank is the count
                // below its position plus its rank among the (few) survivors
                // sharing that position.  (The loop over survivors was 56 %
                // of this kernel's instructions, profiles/r02e_ncu_k_merge_sample.txt.)
                if (keep) atomicAdd(hist + pos, 1);
                __syncwarp();
                int sh = hist[lane];  // -> survivors with pos <= lane
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int t = __shfl_up_sync(kFull, sh, o);
                    if (static_cast<int>(lane) >= o) sh += t;
                }
                const int below = __shfl_sync(kFull, sh, pos > 0 ? pos - 1 : 0);
                int r = pos > 0 ? below : 0;
                if (keep)
                    for (uint32_t g = others & ~dupm; g; g &= g - 1) r += sc[__ffs(g) - 1] < cand;
                __syncwarp();
                outk[lane] = kSentinel;
                outm[lane] = 0u;
                __syncwarp();
                if (in_list && static_cast<int>(lane) + sh < k) {
                    outk[lane + sh] = cur.key;
                    outm[lane + sh] = cur.meta;
                }
                if (keep && pos + r < k) {
                    outk[pos + r] = cand;
                    outm[pos + r] = 3u;  // NEW, from a bucket
                }
                __syncwarp();
                cur.key = outk[lane];
                cur.meta = outm[lane];
            }
            changed = true;
            if (!in_list) cur = Elem{kSentinel, 0u};
            // newcomers that made it into the k-list (oracle's "accepted")
            const uint32_t acc = __ballot_sync(kFull, in_list && (cur.meta >> 1));
            if (lane == 0 && acc && prev_stats) atomicAdd(&prev_stats->accepted, static_cast<unsigned long long>(__popc(acc)));
            cur.meta &= 1u;
            if (lane == 0) G.bcnt[s] = 0;
        }
    }
    if (do_sample) {
        const bool isnew = in_list && (cur.meta & 1u);
        const bool isold = in_list && !(cur.meta & 1u);
        const uint32_t newb = __ballot_sync(kFull, isnew);
        const uint32_t oldb = __ballot_sync(kFull, isold);
        const int rn = __popc(newb & lanemask_lt());
        const int ro = __popc(oldb & lanemask_lt());
        const uint32_t id = key_id(cur.key);
        // the count's old value is the sample's slot in the reverse CSR (one
        // GPU; a distributed refine sends the forward samples to the targets'
        // owners instead, S.fpos == nullptr)
        if (isnew && rn < p) {
            S.fwd[static_cast<size_t>(s) * p + rn] = id;
            if (S.fpos) S.fpos[static_cast<size_t>(s) * p + rn] = atomicAdd(S.rcnt + id, 1u);
            cur.meta &= ~1u;  // "Mark all sampled neighbors as OLD"
        }
        if (isold && ro < p) {
            S.fwd[static_cast<size_t>(D.n) * p + static_cast<size_t>(s) * p + ro] = id;
            if (S.fpos)
                S.fpos[static_cast<size_t>(D.n) * p + static_cast<size_t>(s) * p + ro] = atomicAdd(S.rcnt + D.n + id, 1u);
        }
        if (lane == 0) {
            S.fcnt[2 * s] = static_cast<uint8_t>(min(__popc(newb), p));
            S.fcnt[2 * s + 1] = static_cast<uint8_t>(min(__popc(oldb), p));
        }
    }
    if (changed && in_list) G.keys[static_cast<size_t>(s) * k + lane] = cur.key;
    const uint32_t nm = __ballot_sync(kFull, in_list && (cur.meta & 1u));
    if (lane == 0) G.newmask[s] = nm;
    if (static_cast<int>(lane) == k - 1) G.kth[s] = cur.key;
}

// ------------------------------------------------- CSR offsets
// Exclusive scans (u64) of three per-node counts into S.off[3][n+1]:
//   channel 0/1: reverse NEW / OLD counts (CSR of the reverse appends)
//   channel 2  : bucket capacity of target t, an exact upper bound of the
//                candidates t can receive this iteration: t is in G_new(x)
//                only if x in R_new(t) or x in F_new(t), and gets <= 2 keys
//                from such a join; in G_old(x) only if x in R_old(t) or
//                F_old(t), <= 1 key (Alg. 1 lines 12-31).
// Three phases, 1024 items per block.
constexpr int kScanBlock = 1024;

__device__ __forceinline__ uint64_t block_inclusive_scan(uint64_t v, uint64_t* warp_tot) {
    const uint32_t lane = lane_id(), w = threadIdx.x >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint64_t t = __shfl_up_sync(kFull, v, o);
        if (lane >= static_cast<uint32_t>(o)) v += t;
    }
    if (lane == 31) warp_tot[w] = v;
    __syncthreads();
    if (w == 0) {
        uint64_t x = lane < (blockDim.x >> 5) ? warp_tot[lane] : 0ull;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint64_t t = __shfl_up_sync(kFull, x, o);
            if (lane >= static_cast<uint32_t>(o)) x += t;
        }
        warp_tot[lane] = x;
    }
    __syncthreads();
    if (w > 0) v += warp_tot[w - 1];
    return v;
}

__device__ __forceinline__ uint64_t scan_item(const Samples& S, int64_t n, int f, int64_t i) {
    if (i >= n) return 0ull;
    if (f < 2) return S.rcnt[f * n + i];
    return 2ull * (S.rcnt[i] + S.fcnt[2 * i]) + S.rcnt[n + i] + S.fcnt[2 * i + 1];
}

__global__ void k_scan_reduce(Samples S, int64_t n, int64_t nblk) {
    __shared__ uint64_t wt[32];
    const int f = blockIdx.y;
    const int64_t i = static_cast<int64_t>(blockIdx.x) * kScanBlock + threadIdx.x;
    const uint64_t v = block_inclusive_scan(scan_item(S, n, f, i), wt);
    if (threadIdx.x == kScanBlock - 1) S.bsum[f * nblk + blockIdx.x] = v;
}

__global__ void k_scan_bsums(uint64_t* bsum, int64_t nblk) {
    __shared__ uint64_t wt[32];
    uint64_t* b = bsum + blockIdx.x * nblk;
    const int64_t per = (nblk + kScanBlock - 1) / kScanBlock;
    const int64_t lo = threadIdx.x * per, hi = min(nblk, lo + per);
    uint64_t sum = 0;
    for (int64_t i = lo; i < hi; ++i) sum += b[i];
    const uint64_t incl = block_inclusive_scan(sum, wt);
    uint64_t run = incl - sum;
    for (int64_t i = lo; i < hi; ++i) {
        const uint64_t x = b[i];
        b[i] = run;
        run += x;
    }
}

__global__ void k_scan_final(Samples S, int64_t n, int64_t nblk) {
    __shared__ uint64_t wt[32];
    const int f = blockIdx.y;
    const int64_t i = static_cast<int64_t>(blockIdx.x) * kScanBlock + threadIdx.x;
    const uint64_t v = scan_item(S, n, f, i);
    const uint64_t incl = block_inclusive_scan(v, wt) + S.bsum[f * nblk + blockIdx.x];
    if (i < n) {
        S.off[f * (n + 1) + i] = incl - v;
        if (i == n - 1) S.off[f * (n + 1) + n] = incl;
    }
}

// reverse append of P:149 as a CSR scatter: s goes to the list of every v in
// its forward samples, at the slot its count atomic returned in
// k_merge_sample (no second atomic).  Order inside a list is arbitrary; the
// selection that follows is order-independent (D10).
__global__ void k_rev_scatter(Dims D, Samples S) {
    const int f = blockIdx.y;
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= D.n * D.p) return;
    const int64_t s = i / D.p;
    const int j = static_cast<int>(i - s * D.p);
    if (j >= S.fcnt[2 * s + f]) return;
    const uint32_t v = S.fwd[static_cast<size_t>(f) * D.n * D.p + i];
    const uint32_t pos = S.fpos[static_cast<size_t>(f) * D.n * D.p + i];
    S.rsrc[static_cast<size_t>(f) * S.rstride + S.off[f * (D.n + 1) + v] + pos] = static_cast<uint32_t>(s);
}

// The same, 4 forward samples per thread (p % 4 == 0): the 4 targets' CSR
// offsets are loaded together, so 4 dependent random reads are in flight per
// thread instead of one.
__global__ void k_rev_scatter4(Dims D, Samples S) {
    const int f = blockIdx.y;
    const int64_t i4 = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;  // group of 4 samples
    const int64_t q = D.p >> 2;
    if (i4 >= D.n * q) return;
    const int64_t s = i4 / q;
    const int j0 = static_cast<int>(i4 - s * q) * 4;
    const int fc = S.fcnt[2 * s + f];
    if (j0 >= fc) return;
    const size_t at = static_cast<size_t>(f) * D.n * D.p + static_cast<size_t>(s) * D.p + j0;
    const uint4 v = *reinterpret_cast<const uint4*>(S.fwd + at);
    uint32_t* rs = S.rsrc + static_cast<size_t>(f) * S.rstride;
    const int cnt = min(4, fc - j0);
    const uint32_t src = static_cast<uint32_t>(s);
    const uint4 pos = *reinterpret_cast<const uint4*>(S.fpos + at);
    const uint64_t* off = S.off + f * (D.n + 1);
    uint64_t o0 = off[v.x], o1 = 0, o2 = 0, o3 = 0;
    if (cnt > 1) o1 = off[v.y];
    if (cnt > 2) o2 = off[v.z];
    if (cnt > 3) o3 = off[v.w];
    rs[o0 + pos.x] = src;
    if (cnt > 1) rs[o1 + pos.y] = src;
    if (cnt > 2) rs[o2 + pos.z] = src;
    if (cnt > 3) rs[o3 + pos.w] = src;
}

// sort + dedup one u32 id per lane (0xFFFFFFFF = empty, sorts last); returns
// the unique sorted ids compacted to lanes [0, count) and sets count.
// n: occupied lanes are [0, n) (warp-uniform; the sort runs on blocks of the
// next power of two).  scratch: 32 u32 of per-warp shared memory.
__device__ __forceinline__ uint32_t warp_sort_unique_ids(uint32_t id, int& count, uint32_t* scratch, int n = 32) {
    const uint32_t lane = lane_id();
    const uint32_t x = warp_sort_u32_n(id, n);
    const uint32_t prev = __shfl_sync(kFull, x, (lane + 31) & 31);
    const bool ok = x != 0xFFFFFFFFu && (lane == 0 || x != prev);
    const uint32_t okm = __ballot_sync(kFull, ok);
    count = __popc(okm);
    __syncwarp();
    scratch[lane] = 0xFFFFFFFFu;
    __syncwarp();
    if (ok) scratch[__popc(okm & lanemask_lt())] = x;
    __syncwarp();
    return scratch[lane];
}

// D10 selection for r <= 32 reverse sources (one per lane in `src`): the c
// = cap - fc smallest (Philox x0, s) keys go to lanes [fc, cap) of e.  Fast
// path: sort u32 (x0 with its low 5 bits replaced by the lane), exact as long
// as no two sources share the upper 27 bits of x0 -- then the order by those
// bits is the order by (x0, s).  Returns true (e untouched) when such a tie
// exists; the caller then runs the exact 64-bit path.
__device__ __forceinline__ bool rev_select_ties(uint32_t src, int r, int f, uint32_t tword, int64_t v, uint2 key,
                                                int fc, int c, uint32_t& e) {
    const uint32_t lane = lane_id();
    uint32_t pr = 0xFFFFFFFFu;
    if (static_cast<int>(lane) < r) {
        const uint4 o =
            philox4x32_10(make_uint4(f == 0 ? kTagRevNew : kTagRevOld, tword, src, static_cast<uint32_t>(v)), key);
        pr = (o.x & ~31u) | lane;  // (v: the node's id, D.base + local index)
    }
    pr = warp_sort_u32_n(pr, r);
    const uint32_t prev = __shfl_sync(kFull, pr, (lane + 31) & 31);
    const bool tie = lane > 0 && static_cast<int>(lane) < r && (pr >> 5) == (prev >> 5);
    if (__any_sync(kFull, tie)) return true;
    const int j = static_cast<int>(lane) - fc;
    const bool take = j >= 0 && j < c;
    const uint32_t sel = __shfl_sync(kFull, pr, take ? j : 0);
    const uint32_t id = __shfl_sync(kFull, src, sel & 31u);
    if (take) e = id;
    return false;
}

// One warp per node v: G(v) = sort_unique(F(v) U c smallest-priority reverse
// sources), c = 2p - |F(v)| (P:149 cap 2p with the forward samples counted,
// D8; priority key (Philox(tag, tword, s, v).x, s), D10; P:151 dedup), then
// G_old(v) minus G_new(v) (D11).  Requires 2p <= 32.
__global__ void __launch_bounds__(256, 8) k_rev_select(Dims D, Samples S, uint32_t tword, uint64_t seed) {
    const int64_t v = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (v >= D.n) return;
    const int64_t vid = D.base + v;  // the node's id (the Philox priority word)
    const uint32_t lane = lane_id();
    const uint2 key = seed_key(seed);
    const int p = D.p, cap = D.cap;
    extern __shared__ uint32_t rs_scratch[];  // 64 u32 per warp
    uint32_t* scr = rs_scratch + (threadIdx.x >> 5) * 64;
    uint32_t gnew = 0xFFFFFFFFu;
    int m = 0;
    // both flags' loads up front: counts, CSR bounds, forward row and the
    // first 32 reverse sources (two dependent levels instead of six)
    int fcv[2], rv[2];
    uint64_t o0v[2];
    uint32_t fw[2], pre[2];
#pragma unroll
    for (int f = 0; f < 2; ++f) {
        fcv[f] = S.fcnt[2 * v + f];
        o0v[f] = S.off[f * (D.n + 1) + v];
        rv[f] = static_cast<int>(S.off[f * (D.n + 1) + v + 1] - o0v[f]);
        fw[f] = static_cast<int>(lane) < p ? S.fwd[static_cast<size_t>(f) * D.n * p + static_cast<size_t>(v) * p + lane]
                                           : 0xFFFFFFFFu;
    }
#pragma unroll
    for (int f = 0; f < 2; ++f)
        pre[f] = static_cast<int>(lane) < rv[f] ? S.rsrc[static_cast<size_t>(f) * S.rstride + o0v[f] + lane] : 0xFFFFFFFFu;
#pragma unroll
    for (int f = 0; f < 2; ++f) {
        const int fc = fcv[f];
        const uint32_t* rs = S.rsrc + static_cast<size_t>(f) * S.rstride;
        const uint64_t o0 = o0v[f];
        const int r = rv[f];
        const int c = cap - fc;
        uint32_t e = static_cast<int>(lane) < fc ? fw[f] : 0xFFFFFFFFu;
        if (r <= c) {
            // reverse source j sits in lane j of pre (r <= c <= 32)
            const int j = static_cast<int>(lane) - fc;
            const uint32_t got = __shfl_sync(kFull, pre[f], j >= 0 && j < r ? j : 0);
            if (j >= 0 && j < r) e = got;
        } else if (r <= 32 && !rev_select_ties(pre[f], r, f, tword, vid, key, fc, c, e)) {
            // selected by the 32-bit fast path (no priority ties)
        } else {
            uint64_t best = kSentinel;  // running 32 smallest (prio, s), sorted
            for (int base = 0; base < r; base += 32) {
                uint64_t x = kSentinel;
                if (base + static_cast<int>(lane) < r) {
                    const uint32_t src = base == 0 ? pre[f] : rs[o0 + base + lane];
                    const uint4 o = philox4x32_10(
                        make_uint4(f == 0 ? kTagRevNew : kTagRevOld, tword, src, static_cast<uint32_t>(vid)), key);
                    x = (static_cast<uint64_t>(o.x) << 32) | src;
                }
                x = warp_sort_u64(x);
                if (base == 0) {
                    best = x;
                } else {
                    const uint64_t xr = shfl_u64(x, 31 - lane);
                    best = warp_bitonic_merge_u64(xr < best ? xr : best);
                }
            }
            const int j = static_cast<int>(lane) - fc;
            const uint64_t got = shfl_u64(best, j >= 0 && j < c ? j : 0);
            if (j >= 0 && j < c) e = static_cast<uint32_t>(got);
        }
        int cnt = 0;
        uint32_t u = warp_sort_unique_ids(e, cnt, scr, max(1, fc + min(r, c)));
        if (f == 0) {
            gnew = u;
            m = cnt;
        } else {
            // D11: drop ids that are also NEW samples (binary search in the
            // sorted G_new held in shared memory)
            scr[32 + lane] = gnew;
            __syncwarp();
            int lo = 0;
#pragma unroll
            for (int step = 16; step > 0; step >>= 1)
                if (lo + step <= m && scr[32 + lo + step - 1] < u) lo += step;
            const bool in_new = lo < m && scr[32 + lo] == u;
            const bool keep = static_cast<int>(lane) < cnt && !in_new;
            const uint32_t km = __ballot_sync(kFull, keep);
            cnt = __popc(km);
            __syncwarp();
            scr[lane] = 0xFFFFFFFFu;
            __syncwarp();
            if (keep) scr[__popc(km & lanemask_lt())] = u;
            __syncwarp();
            u = scr[lane];
        }
        if (static_cast<int>(lane) < cnt) S.G[static_cast<size_t>(f) * D.n * cap + static_cast<size_t>(v) * cap + lane] = u;
        if (lane == 0) {
            S.gcnt[2 * v + f] = static_cast<uint8_t>(cnt);
            S.rcnt[f * D.n + v] = 0u;  // counts back to zero for the next iteration
        }
    }
}

// ------------------------------------------------------------------ export
__global__ void k_export(const uint64_t* __restrict__ keys, int64_t total, uint32_t* ids, float* dists) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= total) return;
    const uint64_t kk = keys[i];
    if (ids) ids[i] = key_id(kk);
    if (dists) dists[i] = key_dist(kk);
}

// debug-ABI state conversions: flags u8 [n][k] <-> newmask, plus kth
__global__ void k_state_in(Dims D, Graph G, const uint8_t* __restrict__ flags) {
    const int64_t s = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (s >= D.n) return;
    const uint32_t lane = lane_id();
    const bool in_list = static_cast<int>(lane) < D.k;
    const bool f = in_list && flags[static_cast<size_t>(s) * D.k + lane] != 0;
    const uint32_t nm = __ballot_sync(kFull, f);
    if (lane == 0) {
        G.newmask[s] = nm;
        G.bcnt[s] = 0;
        G.kth[s] = G.keys[static_cast<size_t>(s) * D.k + D.k - 1];
    }
}

__global__ void k_state_out(Dims D, Graph G, uint8_t* flags) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= D.n * D.k) return;
    const int64_t s = i / D.k;
    const int j = static_cast<int>(i - s * D.k);
    flags[i] = static_cast<uint8_t>((G.newmask[s] >> j) & 1u);
}

// Debug copy of G_new/G_old tables into [n][cap] + int32 counts
__global__ void k_samples_out(Dims D, Samples S, uint32_t* Gn, int32_t* cn, uint32_t* Go, int32_t* co) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= D.n * D.cap) return;
    const int64_t v = i / D.cap;
    const int j = static_cast<int>(i - v * D.cap);
    const int m = S.gcnt[2 * v], q = S.gcnt[2 * v + 1];
    Gn[i] = j < m ? S.G[i] : 0u;
    Go[i] = j < q ? S.G[static_cast<size_t>(D.n) * D.cap + i] : 0u;
    if (j == 0) {
        cn[v] = m;
        co[v] = q;
    }
}

// cosine: x^ = x * (1 / sqrtf(sum fmaf(x_i, x_i))) (D6); flags a zero row
__global__ void k_normalize(const float* __restrict__ X, int64_t n, int d, float* Xn, int* bad) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float* x = X + static_cast<size_t>(i) * d;
    float acc = 0.0f;
    for (int j = 0; j < d; ++j) acc = fmaf(x[j], x[j], acc);
    if (!(acc > 0.0f)) {
        atomicExch(bad, 1);
        return;
    }
    const float r = 1.0f / sqrtf(acc);
    float* y = Xn + static_cast<size_t>(i) * d;
    for (int j = 0; j < d; ++j) y[j] = x[j] * r;
}

// option exact_u8: flag any value that is not an integer in [0, 255]
__global__ void k_check_u8(const float* __restrict__ X, int64_t total, int* bad) {
    bool ok = true;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const float v = X[i];
        ok &= (v >= 0.0f && v <= 255.0f && v == rintf(v));
    }
    if (__syncthreads_or(!ok) && threadIdx.x == 0) atomicExch(bad, 1);
}

// chi-square: flag any negative (or NaN) value (D39)
__global__ void k_check_nonneg(const float* __restrict__ X, int64_t total, int* bad) {
    bool ok = true;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        ok &= X[i] >= 0.0f;
    if (__syncthreads_or(!ok) && threadIdx.x == 0) atomicExch(bad, 1);
}

// option exact_u8, fused: one warp per row (d % 4 == 0, 16-B aligned rows)
// checks that every value is an integer in [0, 255], writes the uint8 copy
// and the row's exact squared norm (the tensor-core join's n_c) in one pass
// over the float rows; bad = 1 if any value fails (the copy is then unused)
__global__ void k_to_u8_checked(const float* __restrict__ X, int64_t n, int d, uint8_t* __restrict__ Y,
                                int* __restrict__ sqn, int* bad) {
    const uint32_t lane = lane_id();
    const int64_t w0 = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
    bool ok = true;
    for (int64_t row = w0; row < n; row += nw) {
        const float4* x = reinterpret_cast<const float4*>(X + row * d);
        uchar4* y = reinterpret_cast<uchar4*>(Y + row * d);
        int acc = 0;
        for (int j = static_cast<int>(lane); j < (d >> 2); j += 32) {
            const float4 v = __ldg(x + j);
            ok &= v.x >= 0.0f && v.x <= 255.0f && v.x == rintf(v.x);
            ok &= v.y >= 0.0f && v.y <= 255.0f && v.y == rintf(v.y);
            ok &= v.z >= 0.0f && v.z <= 255.0f && v.z == rintf(v.z);
            ok &= v.w >= 0.0f && v.w <= 255.0f && v.w == rintf(v.w);
            const uchar4 u = make_uchar4(static_cast<uint8_t>(v.x), static_cast<uint8_t>(v.y),
                                         static_cast<uint8_t>(v.z), static_cast<uint8_t>(v.w));
            y[j] = u;
            acc += u.x * u.x + u.y * u.y + u.z * u.z + u.w * u.w;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(kFull, acc, o);
        if (lane == 0) sqn[row] = acc;
    }
    if (__any_sync(kFull, !ok) && lane == 0) atomicExch(bad, 1);
}

__global__ void k_u8_to_f32(const uint8_t* __restrict__ X, int64_t total, float* __restrict__ Y) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        Y[i] = static_cast<float>(X[i]);
}

__global__ void k_to_u8(const float* __restrict__ X, int64_t total, uint8_t* __restrict__ Y) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        Y[i] = static_cast<uint8_t>(X[i]);
}

__global__ void k_philox_test(const uint32_t* __restrict__ ctr, int64_t m, uint64_t seed, uint32_t* out) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= m) return;
    const uint4 c = make_uint4(ctr[4 * i], ctr[4 * i + 1], ctr[4 * i + 2], ctr[4 * i + 3]);
    const uint4 o = philox4x32_10(c, seed_key(seed));
    out[4 * i] = o.x;
    out[4 * i + 1] = o.y;
    out[4 * i + 2] = o.z;
    out[4 * i + 3] = o.w;
}

}  // namespace knng
