// common.cuh -- shared device helpers of the GNND CUDA path (sm_100a).
//
// Nothing here is shared with oracle/: the Philox generator, the canonical
// distance and the warp sorting networks below are this library's own.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace knng {

constexpr uint64_t kSentinel = 0xFFFFFFFFFFFFFFFFull;  // (inf, inf) of Alg. 2
constexpr uint32_t kFull = 0xFFFFFFFFu;

enum : uint32_t { kTagInit = 1, kTagRevNew = 2, kTagRevOld = 3, kTagMergeSeed = 4 };

// key(d, id) = bits(d) << 32 | id  (d >= +0, so u64 order == (d, id) order)
__device__ __forceinline__ uint64_t make_key(float d, uint32_t id) {
    return (static_cast<uint64_t>(__float_as_uint(d)) << 32) | id;
}
__device__ __forceinline__ uint32_t key_id(uint64_t k) { return static_cast<uint32_t>(k); }
__device__ __forceinline__ float key_dist(uint64_t k) {
    return __uint_as_float(static_cast<uint32_t>(k >> 32));
}

// ---------------------------------------------------------------- Philox
// Philox4x32-10 (Salmon et al. SC'11), multipliers 0xD2511F53 / 0xCD9E8D57,
// Weyl key increments 0x9E3779B9 / 0xBB67AE85.
__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 key) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t hi0 = __umulhi(0xD2511F53u, c.x);
        const uint32_t lo0 = 0xD2511F53u * c.x;
        const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z);
        const uint32_t lo1 = 0xCD9E8D57u * c.z;
        c = make_uint4(hi1 ^ c.y ^ key.x, lo1, hi0 ^ c.w ^ key.y, lo0);
        key.x += 0x9E3779B9u;
        key.y += 0xBB67AE85u;
    }
    return c;
}
__device__ __forceinline__ uint2 seed_key(uint64_t seed) {
    return make_uint2(static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32));
}
// uniform integer in [0, N): high 64 bits of (out.y:out.x) * N  (D31)
__device__ __forceinline__ uint64_t uniform_below(uint4 o, uint64_t N) {
    const uint64_t r = (static_cast<uint64_t>(o.y) << 32) | o.x;
    return __umul64hi(r, N);
}

// ---------------------------------------------------------------- warp utils
__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31u; }
__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}
__device__ __forceinline__ uint64_t shfl_u64(uint64_t v, int src) {
    return __shfl_sync(kFull, v, src);
}
__device__ __forceinline__ uint64_t shfl_xor_u64(uint64_t v, int m) {
    return __shfl_xor_sync(kFull, v, m);
}

// Bitonic sorting networks, one value per lane, ascending across lanes.
// Direction by complement: during phase k2 the lanes of a descending block
// hold ~x (bitwise NOT reverses the unsigned order), so every compare-
// exchange of the phase is ascending and the lower lane of a pair keeps the
// minimum: x <- ((o < x) != upper) ? o : x  (taking an equal o is a no-op).
// One u64 compare + two selects per stage (the complement costs two LOPs
// per phase), instead of a per-stage direction test.
__device__ __forceinline__ uint64_t warp_sort_u64(uint64_t x) {
    const uint32_t lane = lane_id();
    uint32_t m_prev = 0;
#pragma unroll
    for (int k2 = 2; k2 <= 32; k2 <<= 1) {
        const uint32_t m = (k2 < 32 && (lane & k2)) ? 0xFFFFFFFFu : 0u;
        const uint32_t t = m ^ m_prev;
        x ^= (static_cast<uint64_t>(t) << 32) | t;
        m_prev = m;
#pragma unroll
        for (int j = k2 >> 1; j > 0; j >>= 1) {
            const uint64_t o = shfl_xor_u64(x, j);
            const bool upper = (lane & j) != 0;
            x = ((o < x) != upper) ? o : x;
        }
    }
    return x;
}
// Bitonic sort of every block of P lanes (P = 2, 4, ..., 32), ascending.
// When only the first P lanes hold data and the rest kSentinel, the whole
// warp is ascending after log2(P) phases instead of 5.
__device__ __forceinline__ uint64_t warp_sort_u64_blocks(uint64_t x, int P) {
    const uint32_t lane = lane_id();
    uint32_t m_prev = 0;
#pragma unroll
    for (int k2 = 2; k2 <= 32; k2 <<= 1) {
        if (k2 > P) break;
        const uint32_t m = (k2 < P && (lane & k2)) ? 0xFFFFFFFFu : 0u;
        const uint32_t t = m ^ m_prev;
        x ^= (static_cast<uint64_t>(t) << 32) | t;
        m_prev = m;
#pragma unroll
        for (int j = k2 >> 1; j > 0; j >>= 1) {
            const uint64_t o = shfl_xor_u64(x, j);
            const bool upper = (lane & j) != 0;
            x = ((o < x) != upper) ? o : x;
        }
    }
    return x;
}
__device__ __forceinline__ uint32_t warp_sort_u32(uint32_t x) {
    const uint32_t lane = lane_id();
    uint32_t m_prev = 0;
#pragma unroll
    for (int k2 = 2; k2 <= 32; k2 <<= 1) {
        const uint32_t m = (k2 < 32 && (lane & k2)) ? 0xFFFFFFFFu : 0u;
        x ^= m ^ m_prev;
        m_prev = m;
#pragma unroll
        for (int j = k2 >> 1; j > 0; j >>= 1) {
            const uint32_t o = __shfl_xor_sync(kFull, x, j);
            x = (lane & j) ? max(o, x) : min(o, x);
        }
    }
    return x;
}
// Bitonic sort of every block of P lanes (P = 2, 4, ..., 32, a compile-time
// constant), ascending: with data in lanes [0, P) and 0xFFFFFFFF above, the
// whole warp is ascending after log2(P) phases instead of 5.
template <int P>
__device__ __forceinline__ uint32_t warp_sort_u32_blocks(uint32_t x) {
    const uint32_t lane = lane_id();
    uint32_t m_prev = 0;
#pragma unroll
    for (int k2 = 2; k2 <= P; k2 <<= 1) {
        const uint32_t m = (k2 < P && (lane & k2)) ? 0xFFFFFFFFu : 0u;
        x ^= m ^ m_prev;
        m_prev = m;
#pragma unroll
        for (int j = k2 >> 1; j > 0; j >>= 1) {
            const uint32_t o = __shfl_xor_sync(kFull, x, j);
            x = (lane & j) ? max(o, x) : min(o, x);
        }
    }
    return x;
}
// ascending sort of lanes [0, n) (0xFFFFFFFF above; n warp-uniform): the
// 16-lane network when the data fits it
__device__ __forceinline__ uint32_t warp_sort_u32_n(uint32_t x, int n) {
    return n <= 16 ? warp_sort_u32_blocks<16>(x) : warp_sort_u32(x);
}
// bitonic sequence across the warp -> ascending
__device__ __forceinline__ uint64_t warp_bitonic_merge_u64(uint64_t x) {
    const uint32_t lane = lane_id();
#pragma unroll
    for (int j = 16; j > 0; j >>= 1) {
        const uint64_t o = shfl_xor_u64(x, j);
        const bool upper = (lane & j) != 0;
        x = ((o < x) != upper) ? o : x;
    }
    return x;
}

// k-NN list update on one warp (D16-D17), branch-free: the list is
// one (key, bits) per lane, ascending, unique, kSentinel-padded; bits =
// bit0 NEW flag | bit1 entered from a bucket.  cand: up to 32 candidate keys
// (any order, repeats allowed, kSentinel = none).  Result: the 32 smallest
// unique keys of the union, ascending; list entries keep their bits,
// newcomers get NEW | from-bucket.  Keys are compared as (key << 1) | origin
// (origin 0 = list, 1 = candidate): dist >= 0 leaves bit 63 free, so the
// shifted order is (dist, id, origin), and duplicates keep the list entry.
// scratch: 32 u64 of per-warp shared memory (compaction by scatter: each
// surviving element writes its rank's slot).
// P: candidates occupy lanes [0, P) only (the rest kSentinel), P a power of 2.
__device__ __forceinline__ void warp_merge_list(uint64_t& L, uint32_t& bits, uint64_t cand, uint64_t* scratch,
                                                int P = 32) {
    const uint32_t lane = lane_id();
    uint64_t x = cand == kSentinel ? kSentinel : ((cand << 1) | 1ull);
    x = warp_sort_u64_blocks(x, P);
    const uint64_t l = L == kSentinel ? kSentinel : (L << 1);
    const uint64_t xr = shfl_u64(x, 31 - lane);  // half-cleaner of l ++ reverse(x)
    uint64_t lo = xr < l ? xr : l;
    uint64_t hi = xr < l ? l : xr;
    lo = warp_bitonic_merge_u64(lo);
    hi = warp_bitonic_merge_u64(hi);
    // dedup: adjacent equal keys (ignoring the origin bit) over lo ++ hi
    const uint64_t lo_prev = shfl_u64(lo, (lane + 31) & 31);
    const uint64_t lo_last = shfl_u64(lo, 31);  // every lane shuffles (no divergent shfl)
    const uint64_t hi_prev_raw = shfl_u64(hi, (lane + 31) & 31);
    const uint64_t hi_prev = lane == 0 ? lo_last : hi_prev_raw;
    const bool lo_ok = lo != kSentinel && (lane == 0 || (lo >> 1) != (lo_prev >> 1));
    const bool hi_ok = hi != kSentinel && (hi >> 1) != (hi_prev >> 1);
    const uint32_t lo_m = __ballot_sync(kFull, lo_ok), hi_m = __ballot_sync(kFull, hi_ok);
    const int nlo = __popc(lo_m);
    // compaction: the j-th surviving element goes to slot j (< 32 kept)
    const int r_lo = __popc(lo_m & lanemask_lt());
    const int r_hi = nlo + __popc(hi_m & lanemask_lt());
    __syncwarp();
    scratch[lane] = kSentinel;
    __syncwarp();
    if (lo_ok) scratch[r_lo] = lo;
    if (hi_ok && r_hi < 32) scratch[r_hi] = hi;
    __syncwarp();
    const uint64_t e = scratch[lane];
    // bits: a list-origin element is the r-th list element kept, r = number
    // of list-origin elements before it (the merge preserves their order)
    const bool is_list = e != kSentinel && !(e & 1ull);
    const int r = __popc(__ballot_sync(kFull, is_list) & lanemask_lt());
    const uint32_t old_bits = __shfl_sync(kFull, bits, r);
    bits = is_list ? old_bits : (e != kSentinel ? 3u : 0u);
    L = e == kSentinel ? kSentinel : (e >> 1);
}

// List update when the candidates are already sorted, unique and disjoint
// from the list (k_merge_sample's pre-filter): y holds (cand << 1) | 1 keys,
// ascending, kSentinel tail.  The 32 smallest of the union are the lower
// half of one half-cleaner -- one bitonic merge, no dedup.  Bits as in
// warp_merge_list.
__device__ __forceinline__ void warp_merge_list_disjoint(uint64_t& L, uint32_t& bits, uint64_t y) {
    const uint32_t lane = lane_id();
    const uint64_t l = L == kSentinel ? kSentinel : (L << 1);
    const uint64_t yr = shfl_u64(y, 31 - lane);
    uint64_t e = yr < l ? yr : l;
    e = warp_bitonic_merge_u64(e);
    const bool is_list = e != kSentinel && !(e & 1ull);
    const int r = __popc(__ballot_sync(kFull, is_list) & lanemask_lt());
    const uint32_t old_bits = __shfl_sync(kFull, bits, r);
    bits = is_list ? old_bits : (e != kSentinel ? 3u : 0u);
    L = e == kSentinel ? kSentinel : (e >> 1);
}

// Element of the list-merge network: key + meta (bit0 = NEW flag, bit1 =
// origin: 0 list, 1 candidate).  Order (key, origin): a list entry sorts in
// front of an equal-key candidate, so dedup keeps the list's flag (D16/D17).
struct Elem {
    uint64_t key;
    uint32_t meta;
};
__device__ __forceinline__ bool elem_less(const Elem& a, const Elem& b) {
    return a.key < b.key || (a.key == b.key && (a.meta >> 1) < (b.meta >> 1));
}
__device__ __forceinline__ Elem shfl_xor_elem(const Elem& e, int m) {
    return Elem{shfl_xor_u64(e.key, m), __shfl_xor_sync(kFull, e.meta, m)};
}
__device__ __forceinline__ Elem shfl_elem(const Elem& e, int src) {
    return Elem{shfl_u64(e.key, src), __shfl_sync(kFull, e.meta, src)};
}
__device__ __forceinline__ Elem warp_sort_elem(Elem x) {
    const uint32_t lane = lane_id();
#pragma unroll
    for (int k2 = 2; k2 <= 32; k2 <<= 1) {
#pragma unroll
        for (int j = k2 >> 1; j > 0; j >>= 1) {
            const Elem o = shfl_xor_elem(x, j);
            const bool up = (lane & k2) == 0;
            const bool lower = (lane & j) == 0;
            const bool o_less = elem_less(o, x);
            const bool take_o = (lower == up) ? o_less : !o_less && (o.key != x.key || o.meta != x.meta);
            if (take_o) x = o;
        }
    }
    return x;
}
// bitonic sequence across the warp -> ascending
__device__ __forceinline__ Elem warp_bitonic_merge_elem(Elem x) {
    const uint32_t lane = lane_id();
#pragma unroll
    for (int j = 16; j > 0; j >>= 1) {
        const Elem o = shfl_xor_elem(x, j);
        const bool lower = (lane & j) == 0;
        const bool o_less = elem_less(o, x);
        if (lower ? o_less : (!o_less && (o.key != x.key || o.meta != x.meta))) x = o;
    }
    return x;
}

// Merge one chunk of up to 32 candidate keys (one per lane, any order, may
// repeat, kSentinel = empty) into a sorted unique list held one entry per
// lane (lanes >= its length hold kSentinel).  Result: the 32 smallest unique
// keys of the union, ascending; list entries keep their NEW flag and origin
// bit, newcomers are NEW with origin = candidate.  scratch: 32 Elem of
// per-warp shared memory.
__device__ __forceinline__ void warp_merge_chunk(Elem& cur, uint64_t cand, Elem* scratch) {
    const uint32_t lane = lane_id();
    Elem b{cand, 3u};  // origin = candidate, NEW
    b = warp_sort_elem(b);
    // half-cleaner of the 64-sequence cur[0..31] ++ reverse(b)
    const Elem br = shfl_elem(b, 31 - lane);
    Elem lo = elem_less(br, cur) ? br : cur;
    Elem hi = elem_less(br, cur) ? cur : br;
    lo = warp_bitonic_merge_elem(lo);
    hi = warp_bitonic_merge_elem(hi);
    // dedup adjacent equal keys over lo[0..31] ++ hi[0..31]
    const uint64_t lo_prev = shfl_u64(lo.key, (lane + 31) & 31);
    const uint64_t lo_last = shfl_u64(lo.key, 31);
    const uint64_t hi_prev_raw = shfl_u64(hi.key, (lane + 31) & 31);
    const uint64_t hi_prev = lane == 0 ? lo_last : hi_prev_raw;
    const bool lo_ok = lo.key != kSentinel && (lane == 0 || lo.key != lo_prev);
    const bool hi_ok = hi.key != kSentinel && hi.key != hi_prev;
    const uint32_t lo_mask = __ballot_sync(kFull, lo_ok);
    const uint32_t hi_mask = __ballot_sync(kFull, hi_ok);
    const int lo_cnt = __popc(lo_mask);
    const int r_lo = __popc(lo_mask & lanemask_lt());
    const int r_hi = lo_cnt + __popc(hi_mask & lanemask_lt());
    __syncwarp();
    scratch[lane] = Elem{kSentinel, 0u};
    __syncwarp();
    if (lo_ok) scratch[r_lo] = lo;
    if (hi_ok && r_hi < 32) scratch[r_hi] = hi;
    __syncwarp();
    cur = scratch[lane];
    __syncwarp();
}

// ---------------------------------------------------------------- distances
// metric template values (= knng_metric)
enum : int { kMetL2 = 0, kMetCos = 1, kMetChi2 = 2 };

__device__ __forceinline__ float chi2_term(float x, float y, float acc) {
    const float t = x - y;
    const float s = x + y;
    const float q = s > 0.0f ? __fdiv_rn(t, s) : 0.0f;
    return fmaf(q, t, acc);
}

// Canonical distances (D5/D6): one thread owns one pair and accumulates the
// dimensions in order 0..d-1: acc = fmaf(x_i - y_i, x_i - y_i, acc).
template <typename T>
struct Canon;

template <>
struct Canon<float> {
    __device__ static __forceinline__ float l2(const float* __restrict__ a,
                                               const float* __restrict__ b, int d) {
        float acc = 0.0f;
        if ((d & 3) == 0 && ((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(b)) & 15) == 0) {
            const float4* a4 = reinterpret_cast<const float4*>(a);
            const float4* b4 = reinterpret_cast<const float4*>(b);
            for (int i = 0; i < (d >> 2); ++i) {
                const float4 x = __ldg(a4 + i), y = __ldg(b4 + i);
                float t;
                t = x.x - y.x; acc = fmaf(t, t, acc);
                t = x.y - y.y; acc = fmaf(t, t, acc);
                t = x.z - y.z; acc = fmaf(t, t, acc);
                t = x.w - y.w; acc = fmaf(t, t, acc);
            }
        } else {
            for (int i = 0; i < d; ++i) {
                const float t = __ldg(a + i) - __ldg(b + i);
                acc = fmaf(t, t, acc);
            }
        }
        return acc;
    }
    // chi-square ("K-Square"), D39: q = t / s (0 when s = 0),
    // acc = fmaf(q, t, acc) in dimension order (IEEE division: no fast math)
    __device__ static __forceinline__ float chi2(const float* __restrict__ a, const float* __restrict__ b, int d) {
        float acc = 0.0f;
        for (int i = 0; i < d; ++i) acc = chi2_term(__ldg(a + i), __ldg(b + i), acc);
        return acc;
    }
    // 1 - <x^, y^> on pre-normalised rows, clamped at +0 (D6)
    __device__ static __forceinline__ float cos(const float* __restrict__ a,
                                                const float* __restrict__ b, int d) {
        float s = 0.0f;
        for (int i = 0; i < d; ++i) s = fmaf(__ldg(a + i), __ldg(b + i), s);
        const float r = 1.0f - s;
        return r > 0.0f ? r : 0.0f;
    }
};

template <>
struct Canon<uint8_t> {
    __device__ static __forceinline__ float l2(const uint8_t* __restrict__ a,
                                               const uint8_t* __restrict__ b, int d) {
        if ((d & 15) == 0 && ((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(b)) & 15) == 0) {
            // integer sums are exact in any order: 16 dims per 128-bit load
            unsigned int acc = 0;
            const uint4* a4 = reinterpret_cast<const uint4*>(a);
            const uint4* b4 = reinterpret_cast<const uint4*>(b);
            for (int i = 0; i < (d >> 4); ++i) {
                const uint4 x = __ldg(a4 + i), y = __ldg(b4 + i);
                uint32_t t;
                t = __vabsdiffu4(x.x, y.x); acc = __dp4a(t, t, acc);
                t = __vabsdiffu4(x.y, y.y); acc = __dp4a(t, t, acc);
                t = __vabsdiffu4(x.z, y.z); acc = __dp4a(t, t, acc);
                t = __vabsdiffu4(x.w, y.w); acc = __dp4a(t, t, acc);
            }
            return static_cast<float>(acc);
        }
        int acc = 0;
        for (int i = 0; i < d; ++i) {
            const int t = static_cast<int>(__ldg(a + i)) - static_cast<int>(__ldg(b + i));
            acc += t * t;
        }
        return static_cast<float>(acc);
    }
};

}  // namespace knng
