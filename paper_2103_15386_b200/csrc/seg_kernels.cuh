// seg_kernels.cuh -- segmented k-NN lists for k = 32 s, s = 2 .. 4 (SURVEY.md
// 8(f) N2; "k-NN list is divided into k / 32 segments.  Each segment
// keeps 32 (the size of a warp) neighbors.  The object v will be inserted
// into the v % (k / 32)-th segment ... As the iteration is completed, all the
// segments of one k-NN list will be merged into one"; reading D40).
//
// Layout: segment-major, keys[x][g][32] (segment g holds ids = g mod s, 32
// entries, ascending), newmask[x][g] (bit j: entry j of segment g is NEW),
// kth[x] = the largest of the s segment maxima (the joins' filter is then
// loose; the per-segment merge below is exact, D17).  The "merged" list of
// the union in (dist, id) order -- is what sampling (first p NEW /
// OLD, D7) and the export read: every entry's position in it is its
// rank in its own segment plus, per other segment, the number of keys below
// it (a 5-step binary search in shared memory).  One warp per node.
#pragma once
#include "graph_kernels.cuh"

namespace knng {

template <typename T, int MET>
__device__ __forceinline__ float canon_dist(const T* __restrict__ X, const float* __restrict__ Xn, int d, int64_t a,
                                            int64_t b) {
    if constexpr (MET == kMetCos) return Canon<float>::cos(Xn + static_cast<size_t>(a) * d, Xn + static_cast<size_t>(b) * d, d);
    if constexpr (MET == kMetChi2)
        return Canon<float>::chi2(reinterpret_cast<const float*>(X) + static_cast<size_t>(a) * d,
                                  reinterpret_cast<const float*>(X) + static_cast<size_t>(b) * d, d);
    return Canon<T>::l2(X + static_cast<size_t>(a) * d, X + static_cast<size_t>(b) * d, d);
}

// number of keys < e in the ascending 32-key segment seg (shared memory)
__device__ __forceinline__ int seg_count_below(const uint64_t* seg, uint64_t e) {
    int pos = 0;
#pragma unroll
    for (int step = 16; step > 0; step >>= 1)
        if (seg[pos + step - 1] < e) pos += step;
    return pos + (seg[pos] < e ? 1 : 0);  // pos <= 31 here; 32 if all below
}
__device__ __forceinline__ uint32_t low_bits(int c) { return c >= 32 ? 0xFFFFFFFFu : ((1u << c) - 1u); }

// Init (Alg. 1 lines 1-4 with D40): segment g draws 32 distinct ids of the
// residue class g mod s (self excluded) in counter order from
// Philox(INIT, x, j | g << 24, x >> 32); canonical distances; sorted.
template <typename T, int MET, int SEG>
__global__ void k_init_seg(const T* __restrict__ X, const float* __restrict__ Xn, Dims D, uint64_t seed, Graph G) {
    const int64_t x = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (x >= D.n) return;
    const uint32_t lane = lane_id();
    const uint2 key = seed_key(seed);
    extern __shared__ uint32_t iseg_scratch[];
    uint32_t* scr = iseg_scratch + (threadIdx.x >> 5) * 32;
    uint64_t kmax = 0;
    for (int g = 0; g < SEG; ++g) {
        const int64_t M = (D.n - g + SEG - 1) / SEG;
        const bool self_in = (x % SEG) == g;
        const uint64_t range = static_cast<uint64_t>(M - (self_in ? 1 : 0));
        uint32_t chosen = 0xFFFFFFFFu;
        int cnt = 0;
        for (uint32_t j0 = 0; cnt < 32; j0 += 32) {
            const uint4 o = philox4x32_10(make_uint4(kTagInit, static_cast<uint32_t>(x), (j0 + lane) | (static_cast<uint32_t>(g) << 24),
                                                     static_cast<uint32_t>(static_cast<uint64_t>(x) >> 32)),
                                          key);
            uint64_t v = static_cast<uint64_t>(g) + static_cast<uint64_t>(SEG) * uniform_below(o, range);
            if (self_in && v >= static_cast<uint64_t>(x)) v += SEG;
            const uint32_t vv = static_cast<uint32_t>(v);
            bool dup = false;
            for (int t = 0; t < cnt; ++t) dup |= (__shfl_sync(kFull, chosen, t) == vv);
            dup |= (__match_any_sync(kFull, vv) & lanemask_lt()) != 0u;
            const uint32_t acc = __ballot_sync(kFull, !dup);
            const int slot = cnt + __popc(acc & lanemask_lt());
            __syncwarp();
            if (!dup && slot < 32) scr[slot] = vv;
            __syncwarp();
            const int nc = min(32, cnt + __popc(acc));
            if (static_cast<int>(lane) >= cnt && static_cast<int>(lane) < nc) chosen = scr[lane];
            cnt = nc;
        }
        uint64_t kk = make_key(canon_dist<T, MET>(X, Xn, D.d, x, chosen), chosen);
        kk = warp_sort_u64(kk);
        G.keys[static_cast<size_t>(x) * D.k + g * 32 + lane] = kk;
        const uint64_t top = shfl_u64(kk, 31);
        kmax = top > kmax ? top : kmax;
    }
    if (lane < SEG) G.newmask[x * SEG + lane] = kFull;
    if (lane == 0) G.kth[x] = kmax;
}

// List update + sampling (as k_merge_sample, per segment, D40).
template <int SEG>
__global__ void __launch_bounds__(256) k_merge_sample_seg(Dims D, Graph G, Samples S, int do_merge, int do_sample,
                                                          DevStats* __restrict__ prev_stats) {
    const int64_t x = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (x >= D.n) return;
    const uint32_t lane = lane_id();
    const int p = D.p;
    extern __shared__ uint64_t mseg_smem[];  // per warp: SEG * 32 keys + 32 scratch
    uint64_t* sk = mseg_smem + (threadIdx.x >> 5) * (SEG * 32 + 32);
    uint64_t* scr = sk + SEG * 32;
    uint64_t L[SEG];
    uint32_t bits[SEG];
#pragma unroll
    for (int g = 0; g < SEG; ++g) {
        L[g] = G.keys[static_cast<size_t>(x) * D.k + g * 32 + lane];
        bits[g] = (G.newmask[x * SEG + g] >> lane) & 1u;
    }
    unsigned long long acc = 0;
    if (G.imask) {  // locked immediate update: entries that entered last iteration
#pragma unroll
        for (int g = 0; g < SEG; ++g) acc += __popc(G.imask[x * SEG + g]);
        __syncwarp();
        if (lane < SEG) G.imask[x * SEG + lane] = 0;
    }
    bool changed = false;
    if (do_merge) {
        const uint32_t c = G.bcnt[x];
        if (c > 0) {
            const uint64_t* bk = G.bucket + G.boff[x];
            for (uint32_t base = 0; base < c; base += 32) {
                const uint64_t cand = (base + lane < c) ? bk[base + lane] : kSentinel;
#pragma unroll
                for (int g = 0; g < SEG; ++g) {
                    const uint64_t cg = (cand != kSentinel && key_id(cand) % SEG == static_cast<uint32_t>(g)) ? cand : kSentinel;
                    const uint64_t gmax = shfl_u64(L[g], 31);
                    if (__any_sync(kFull, cg < gmax))  // else no key of the chunk can enter segment g
                        warp_merge_list(L[g], bits[g], cg, scr);
                }
            }
#pragma unroll
            for (int g = 0; g < SEG; ++g) {
                acc += __popc(__ballot_sync(kFull, bits[g] & 2u));
                bits[g] &= 1u;
            }
            changed = true;
            if (lane == 0) G.bcnt[x] = 0;
        }
    }
    if (lane == 0 && acc && prev_stats) atomicAdd(&prev_stats->accepted, acc);
    if (do_sample) {
        uint32_t nw[SEG], ow[SEG];
#pragma unroll
        for (int g = 0; g < SEG; ++g) {
            sk[g * 32 + lane] = L[g];
            nw[g] = __ballot_sync(kFull, L[g] != kSentinel && (bits[g] & 1u));
            ow[g] = __ballot_sync(kFull, L[g] != kSentinel && !(bits[g] & 1u));
        }
        __syncwarp();
        int tn = 0, to = 0;
#pragma unroll
        for (int g = 0; g < SEG; ++g) {
            tn += __popc(nw[g]);
            to += __popc(ow[g]);
        }
#pragma unroll
        for (int g = 0; g < SEG; ++g) {
            // ranks among the NEW / OLD entries of the merged list (D7)
            int rn = __popc(nw[g] & lanemask_lt()), ro = __popc(ow[g] & lanemask_lt());
#pragma unroll
            for (int h = 0; h < SEG; ++h) {
                if (h == g) continue;
                const int below = seg_count_below(sk + h * 32, L[g]);
                rn += __popc(nw[h] & low_bits(below));
                ro += __popc(ow[h] & low_bits(below));
            }
            const uint32_t id = key_id(L[g]);
            if (((nw[g] >> lane) & 1u) && rn < p) {
                S.fwd[static_cast<size_t>(x) * p + rn] = id;
                if (S.fpos) S.fpos[static_cast<size_t>(x) * p + rn] = atomicAdd(S.rcnt + id, 1u);
                bits[g] &= ~1u;  // "Mark all sampled neighbors as OLD"
            }
            if (((ow[g] >> lane) & 1u) && ro < p) {
                S.fwd[static_cast<size_t>(D.n) * p + static_cast<size_t>(x) * p + ro] = id;
                if (S.fpos)
                    S.fpos[static_cast<size_t>(D.n) * p + static_cast<size_t>(x) * p + ro] = atomicAdd(S.rcnt + D.n + id, 1u);
            }
        }
        if (lane == 0) {
            S.fcnt[2 * x] = static_cast<uint8_t>(min(tn, p));
            S.fcnt[2 * x + 1] = static_cast<uint8_t>(min(to, p));
        }
    }
    uint64_t kmax = 0;
#pragma unroll
    for (int g = 0; g < SEG; ++g) {
        if (changed) G.keys[static_cast<size_t>(x) * D.k + g * 32 + lane] = L[g];
        const uint32_t nm = __ballot_sync(kFull, bits[g] & 1u);
        if (lane == 0) G.newmask[x * SEG + g] = nm;
        const uint64_t top = shfl_u64(L[g], 31);
        kmax = top > kmax ? top : kmax;
    }
    if (lane == 0) G.kth[x] = kmax;
}

// The merged list: ids / dists [n][k] ascending, optional u8 flags.
template <int SEG>
__global__ void k_export_seg(Dims D, Graph G, uint32_t* ids, float* dists, uint64_t* keys_out, uint8_t* flags_out) {
    const int64_t x = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (x >= D.n) return;
    const uint32_t lane = lane_id();
    extern __shared__ uint64_t eseg_smem[];
    uint64_t* sk = eseg_smem + (threadIdx.x >> 5) * (SEG * 32);
    uint64_t L[SEG];
#pragma unroll
    for (int g = 0; g < SEG; ++g) {
        L[g] = G.keys[static_cast<size_t>(x) * D.k + g * 32 + lane];
        sk[g * 32 + lane] = L[g];
    }
    __syncwarp();
#pragma unroll
    for (int g = 0; g < SEG; ++g) {
        int pos = static_cast<int>(lane);
#pragma unroll
        for (int h = 0; h < SEG; ++h)
            if (h != g) pos += seg_count_below(sk + h * 32, L[g]);
        const size_t o = static_cast<size_t>(x) * D.k + pos;
        if (ids) ids[o] = key_id(L[g]);
        if (dists) dists[o] = key_dist(L[g]);
        if (keys_out) keys_out[o] = L[g];
        if (flags_out) flags_out[o] = static_cast<uint8_t>((G.newmask[x * SEG + g] >> lane) & 1u);
    }
}

// debug ABI: merged keys + u8 flags [n][k] (ascending) -> segment-major state
template <int SEG>
__global__ void k_state_in_seg(Dims D, Graph G, const uint64_t* __restrict__ keys_in, const uint8_t* __restrict__ flags) {
    const int64_t x = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (x >= D.n) return;
    const uint32_t lane = lane_id();
    extern __shared__ uint64_t sseg_smem[];
    uint64_t* sk = sseg_smem + (threadIdx.x >> 5) * (SEG * 32);
    uint32_t* sf = reinterpret_cast<uint32_t*>(sseg_smem + (blockDim.x >> 5) * SEG * 32) + (threadIdx.x >> 5) * SEG;
    if (lane < SEG) sf[lane] = 0;
    int fill[SEG];
#pragma unroll
    for (int g = 0; g < SEG; ++g) fill[g] = 0;
    __syncwarp();
    for (int c = 0; c < SEG; ++c) {  // merged list, 32 entries at a time
        const uint64_t e = keys_in[static_cast<size_t>(x) * D.k + c * 32 + lane];
        const bool nw = flags[static_cast<size_t>(x) * D.k + c * 32 + lane] != 0;
        const int g0 = static_cast<int>(key_id(e) % SEG);
#pragma unroll
        for (int g = 0; g < SEG; ++g) {
            const uint32_t m = __ballot_sync(kFull, g0 == g);
            if (g0 == g) {
                const int slot = fill[g] + __popc(m & lanemask_lt());
                sk[g * 32 + slot] = e;
                if (nw) atomicOr(sf + g, 1u << slot);
            }
            fill[g] += __popc(m);
        }
    }
    __syncwarp();
    uint64_t kmax = 0;
#pragma unroll
    for (int g = 0; g < SEG; ++g) {
        const uint64_t e = sk[g * 32 + lane];
        G.keys[static_cast<size_t>(x) * D.k + g * 32 + lane] = e;
        const uint64_t top = shfl_u64(e, 31);
        kmax = top > kmax ? top : kmax;
    }
    if (lane < SEG) G.newmask[x * SEG + lane] = sf[lane];
    if (lane == 0) {
        G.bcnt[x] = 0;
        G.kth[x] = kmax;
    }
}

}  // namespace knng
