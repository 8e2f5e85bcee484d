// order_kernels.cuh -- processing order of the local joins (a performance
// device only; results do not depend on it).
//
// The joins of one iteration read only G_new/G_old and the vectors, and the
// update is bulk-synchronous and order-independent (D17), so the join kernel
// may visit the nodes in any order.  Visiting nodes whose vectors are close
// one after another makes their sample sets overlap: the same rows are
// gathered by many CTAs at about the same time and are served from L2.
// The order: a 16-bit random-projection code per node -- bit j = sign of
// <x - mean, r_j> with r_j a fixed pseudo-random +-1 vector -- and a counting
// sort by code (order inside a code bucket is whatever the atomics give;
// irrelevant for the result).
#pragma once
#include "common.cuh"

namespace knng {

constexpr int kOrderBits = 16;
constexpr int kOrderBuckets = 1 << kOrderBits;

__device__ __forceinline__ float order_sign(int j, int i) {
    // +-1, a fixed function of (direction j, dimension i)
    uint32_t h = static_cast<uint32_t>(j) * 0x9E3779B1u ^ static_cast<uint32_t>(i) * 0x85EBCA77u;
    h ^= h >> 15;
    h *= 0x2C1B3C6Du;
    h ^= h >> 12;
    return (h & 1u) ? 1.0f : -1.0f;
}

// column sums (for the mean): block-local partial sums, then one atomic per
// dimension and block
template <typename T>
__global__ void k_order_colsum(const T* __restrict__ X, int64_t n, int d, float* __restrict__ sum) {
    const int64_t per = (n + gridDim.x - 1) / gridDim.x;
    const int64_t r0 = blockIdx.x * per, r1 = min(n, r0 + per);
    for (int i = threadIdx.x; i < d; i += blockDim.x) {
        float acc = 0.0f;
        for (int64_t r = r0; r < r1; ++r) acc += static_cast<float>(X[r * d + i]);
        atomicAdd(sum + i, acc);
    }
}

// code of every node + bucket histogram (d <= kOrderMaxD: the directions
// and the mean live in shared memory)
constexpr int kOrderMaxD = 128;
template <typename T>
__global__ void k_order_code(const T* __restrict__ X, int64_t n, int d, const float* __restrict__ sum,
                             uint32_t* __restrict__ code, uint32_t* __restrict__ hist) {
    __shared__ float sg[kOrderBits][kOrderMaxD];
    __shared__ float mu[kOrderMaxD];
    const float inv = 1.0f / static_cast<float>(n);
    for (int e = threadIdx.x; e < kOrderBits * d; e += blockDim.x) sg[e / d][e % d] = order_sign(e / d, e % d);
    for (int i = threadIdx.x; i < d; i += blockDim.x) mu[i] = sum[i] * inv;
    __syncthreads();
    const int64_t x = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (x >= n) return;
    float proj[kOrderBits];
#pragma unroll
    for (int j = 0; j < kOrderBits; ++j) proj[j] = 0.0f;
    const T* row = X + x * d;
    for (int i = 0; i < d; ++i) {
        const float v = static_cast<float>(row[i]) - mu[i];
#pragma unroll
        for (int j = 0; j < kOrderBits; ++j) proj[j] = fmaf(sg[j][i], v, proj[j]);
    }
    uint32_t c = 0;
#pragma unroll
    for (int j = 0; j < kOrderBits; ++j) c |= (proj[j] > 0.0f ? 1u : 0u) << j;
    code[x] = c;
    atomicAdd(hist + c, 1u);
}

// exclusive scan of the 65536 bucket counts in place (one block of 256)
__global__ void __launch_bounds__(256) k_order_scan(uint32_t* __restrict__ hist) {
    __shared__ uint32_t part[256];
    constexpr int per = kOrderBuckets / 256;
    const int t = threadIdx.x;
    uint32_t s = 0;
    for (int i = 0; i < per; ++i) s += hist[t * per + i];
    part[t] = s;
    __syncthreads();
    for (int o = 1; o < 256; o <<= 1) {
        const uint32_t v = t >= o ? part[t - o] : 0u;
        __syncthreads();
        part[t] += v;
        __syncthreads();
    }
    uint32_t run = part[t] - s;
    for (int i = 0; i < per; ++i) {
        const uint32_t c = hist[t * per + i];
        hist[t * per + i] = run;
        run += c;
    }
}

__global__ void k_order_scatter(const uint32_t* __restrict__ code, int64_t n, uint32_t* __restrict__ cursor,
                                uint32_t* __restrict__ perm) {
    const int64_t x = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (x >= n) return;
    perm[atomicAdd(cursor + code[x], 1u)] = static_cast<uint32_t>(x);
}

}  // namespace knng
