// Microbenchmark of the float join's consumer inner loop in isolation:
// 4x4 (and 4x8) register blocks of packed FP32x2 canonical L2 steps reading
// the pair-interleaved stage layout of join_ws.cuh from shared memory, no
// barriers.  Reports lane-ops/s (2 per pair-dim) against the 36 T peak.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned long long f2_l2(float a, unsigned long long b, unsigned long long acc) {
    unsigned long long r;
    asm("{\n\t.reg .b64 aa, tt;\n\tmov.b64 aa, {%1, %1};\n\tsub.rn.f32x2 tt, aa, %2;\n\tfma.rn.f32x2 %0, tt, tt, %3;\n\t}"
        : "=l"(r) : "f"(a), "l"(b), "l"(acc));
    return r;
}
constexpr int G = 132;
template <int NCB>  // column blocks of 4 per thread
__global__ void __launch_bounds__(256) k(float* out, int reps, int stride) {
    __shared__ __align__(16) float st[64 * G];
    for (int i = threadIdx.x; i < 64 * G; i += 256) st[i] = i * 1e-4f;
    __syncthreads();
    const int ct = threadIdx.x;
    const int gA = ct % 64, gB0 = (ct * stride) % 64;
    unsigned long long acc[4][2 * NCB];
    for (int r = 0; r < 4; ++r) for (int c = 0; c < 2 * NCB; ++c) acc[r][c] = 0;
    for (int rep = 0; rep < reps; ++rep) {
        const float* A = st + ((gA + rep) & 63) * G;
#pragma unroll
        for (int c = 0; c < 16; ++c) {
            const int pos = (((c & 1) << 3) | (c >> 1)) * 4;
            const float4 a01 = *reinterpret_cast<const float4*>(A + pos);
            const float4 a23 = *reinterpret_cast<const float4*>(A + 64 + pos);
            ulonglong2 b[NCB][2];
#pragma unroll
            for (int cb = 0; cb < NCB; ++cb) {
                const float* B = st + ((gB0 + cb * 9 + rep * 3) & 63) * G;
                b[cb][0] = *reinterpret_cast<const ulonglong2*>(B + pos);
                b[cb][1] = *reinterpret_cast<const ulonglong2*>(B + 64 + pos);
            }
            const float ar[2][4] = {{a01.x, a01.y, a23.x, a23.y}, {a01.z, a01.w, a23.z, a23.w}};
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
                for (int r = 0; r < 4; ++r)
#pragma unroll
                    for (int cb = 0; cb < NCB; ++cb) {
                        const unsigned long long p0 = h ? b[cb][0].y : b[cb][0].x, p1 = h ? b[cb][1].y : b[cb][1].x;
                        acc[r][2 * cb] = f2_l2(ar[h][r], p0, acc[r][2 * cb]);
                        acc[r][2 * cb + 1] = f2_l2(ar[h][r], p1, acc[r][2 * cb + 1]);
                    }
        }
    }
    float s = 0;
    for (int r = 0; r < 4; ++r) for (int c = 0; c < 2 * NCB; ++c) s += __uint_as_float((unsigned)acc[r][c]);
    out[blockIdx.x * 256 + threadIdx.x] = s;
}
int main() {
    float* out; cudaMalloc(&out, 148 * 4 * 256 * sizeof(float));
    const int reps = 4000;
    for (int ncb = 1; ncb <= 2; ++ncb)
        for (int ctas = 1; ctas <= 3; ++ctas)
            for (int stride = 1; stride <= 7; stride += 6) {
                cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
                auto go = [&]() { if (ncb == 1) k<1><<<148 * ctas, 256>>>(out, reps, stride); else k<2><<<148 * ctas, 256>>>(out, reps, stride); };
                go(); cudaEventRecord(e0); go(); cudaEventRecord(e1); cudaEventSynchronize(e1);
                float ms; cudaEventElapsedTime(&ms, e0, e1);
                double ops = 148.0 * ctas * 256 * reps * 16 * 2 /*dims*/ * 16 * ncb /*pairs*/ * 2;
                printf("4x%d block, %d CTA(s)/SM (8 warps each), B stride %d: %.3f ms  %.1f T lane-ops/s (%.0f%% of 36)\n",
                       4 * ncb, ctas, stride, ms, ops / ms / 1e9, ops / ms / 1e9 / 36 * 100);
            }
    return 0;
}
