// eval_kernels.cuh -- exact k-NN by exhaustive scan for recall@10
// ground truth (Eq. 4).  Not on the timed path.
//
// CTA = W warps; each warp owns QW queries (lane-parallel over data points).
// A tile of 32 data rows is staged into shared memory (row stride odd in
// 4-byte words: conflict-free lane-strided reads); each lane computes the
// canonical distance (D5/D6) of its data row to each of the warp's queries,
// and a warp merges the 32 candidate keys into each query's running top-kq
// whenever one of them beats the current kq-th key.
#pragma once
#include "graph_kernels.cuh"

namespace knng {

constexpr int kBfQPerWarp = 4;

template <typename T>
__host__ __device__ inline int bf_stride_elems(int d) {
    // row stride in elements with an odd number of 4-byte words
    const int bytes = d * static_cast<int>(sizeof(T));
    int words = (bytes + 3) / 4;
    if ((words & 1) == 0) words += 1;
    return words * 4 / static_cast<int>(sizeof(T));
}

template <typename T, int MET>
__global__ void k_bruteforce(const T* __restrict__ X, const float* __restrict__ Xn, int64_t n, int d,
                             const int64_t* __restrict__ queries, int64_t nq, int kq, uint64_t* out) {
    using E = typename std::conditional<MET == kMetCos, float, T>::type;
    const E* __restrict__ V = MET == kMetCos ? reinterpret_cast<const E*>(Xn) : reinterpret_cast<const E*>(X);
    extern __shared__ __align__(16) unsigned char bf_smem[];
    const int W = blockDim.x >> 5;
    const int stride = bf_stride_elems<E>(d);
    E* tile = reinterpret_cast<E*>(bf_smem);                                      // [32][stride]
    E* qv = tile + 32 * stride;                                                    // [W*QW][stride]
    Elem* scratch = reinterpret_cast<Elem*>(qv + static_cast<size_t>(W) * kBfQPerWarp * stride);  // [W][32]
    const int warp = threadIdx.x >> 5;
    const uint32_t lane = lane_id();
    const int64_t q0 = (static_cast<int64_t>(blockIdx.x) * W + warp) * kBfQPerWarp;
    Elem* scr = scratch + warp * 32;

    // stage this warp's query rows
    for (int qi = 0; qi < kBfQPerWarp; ++qi) {
        const int64_t qq = q0 + qi;
        for (int j = lane; j < d; j += 32)
            qv[(warp * kBfQPerWarp + qi) * stride + j] = qq < nq ? V[static_cast<size_t>(queries[qq]) * d + j] : E(0);
    }
    int64_t qid[kBfQPerWarp];
    for (int qi = 0; qi < kBfQPerWarp; ++qi) qid[qi] = (q0 + qi < nq) ? queries[q0 + qi] : -1;
    Elem best[kBfQPerWarp];
    for (int qi = 0; qi < kBfQPerWarp; ++qi) best[qi] = Elem{kSentinel, 0u};

    for (int64_t base = 0; base < n; base += 32) {
        __syncthreads();
        for (int idx = threadIdx.x; idx < 32 * d; idx += blockDim.x) {
            const int r = idx / d, j = idx - r * d;
            const int64_t row = base + r;
            tile[r * stride + j] = row < n ? V[static_cast<size_t>(row) * d + j] : E(0);
        }
        __syncthreads();
        const int64_t pt = base + lane;
        const E* prow = tile + lane * stride;
#pragma unroll
        for (int qi = 0; qi < kBfQPerWarp; ++qi) {
            if (qid[qi] < 0) continue;  // warp-uniform
            const E* qrow = qv + (warp * kBfQPerWarp + qi) * stride;
            float dist;
            if constexpr (MET == kMetCos) {
                float s = 0.0f;
                for (int j = 0; j < d; ++j) s = fmaf(qrow[j], prow[j], s);
                const float r = 1.0f - s;
                dist = r > 0.0f ? r : 0.0f;
            } else if constexpr (MET == kMetChi2) {
                float acc = 0.0f;
                for (int j = 0; j < d; ++j) acc = chi2_term(qrow[j], prow[j], acc);
                dist = acc;
            } else if constexpr (std::is_same<E, float>::value) {
                float acc = 0.0f;
                for (int j = 0; j < d; ++j) {
                    const float t = qrow[j] - prow[j];
                    acc = fmaf(t, t, acc);
                }
                dist = acc;
            } else {
                int acc = 0;
                for (int j = 0; j < d; ++j) {
                    const int t = static_cast<int>(qrow[j]) - static_cast<int>(prow[j]);
                    acc += t * t;
                }
                dist = static_cast<float>(acc);
            }
            const uint64_t key = (pt < n && pt != qid[qi]) ? make_key(dist, static_cast<uint32_t>(pt)) : kSentinel;
            const uint64_t worst = shfl_u64(best[qi].key, kq - 1);
            if (__ballot_sync(kFull, key < worst)) {
                warp_merge_chunk(best[qi], key, scr);
                if (static_cast<int>(lane) >= kq) best[qi] = Elem{kSentinel, 0u};
            }
        }
    }
    for (int qi = 0; qi < kBfQPerWarp; ++qi)
        if (qid[qi] >= 0 && static_cast<int>(lane) < kq) out[(q0 + qi) * kq + lane] = best[qi].key;
}

}  // namespace knng
