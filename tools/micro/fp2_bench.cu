// Microbenchmark: scalar FP32 vs packed FP32x2 (FADD2/FFMA2) throughput on
// one B200 (lane-ops per second), for the canonical L2 step pattern
// t = a - b; acc = fma(t, t, acc).  nvcc -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned long long f2_l2(float a, unsigned long long b, unsigned long long acc) {
    unsigned long long r;
    asm volatile("{\n\t.reg .b64 aa, tt;\n\tmov.b64 aa, {%1, %1};\n\tsub.rn.f32x2 tt, aa, %2;\n\tfma.rn.f32x2 %0, tt, tt, %3;\n\t}"
        : "=l"(r) : "f"(a), "l"(b), "l"(acc));
    return r;
}
__device__ __forceinline__ unsigned long long f2_fma(unsigned long long a, unsigned long long b, unsigned long long acc) {
    unsigned long long r;
    asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(acc));
    return r;
}
template <int MODE>
__global__ void k(float* out, int iters, float s) {
    float a = threadIdx.x * 1e-3f, b0 = s, b1 = s * 2;
    if (MODE == 0) {  // scalar L2 step: 16 chains
        float acc[16];
        for (int i = 0; i < 16; ++i) acc[i] = 0.f;
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int i = 0; i < 16; ++i) { float t = a - (b0 + i); acc[i] = __fmaf_rn(t, t, acc[i]); }
            a += 1e-7f;
        }
        float r = 0; for (int i = 0; i < 16; ++i) r += acc[i];
        out[blockIdx.x * blockDim.x + threadIdx.x] = r;
    } else if (MODE == 1) {  // packed L2 step: 8 packed chains = 16 lanes
        unsigned long long acc[8], bb[8];
        for (int i = 0; i < 8; ++i) { acc[i] = 0; float x = b0 + i, y = b1 + i; asm("mov.b64 %0, {%1,%2};" : "=l"(bb[i]) : "f"(x), "f"(y)); }
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int i = 0; i < 8; ++i) acc[i] = f2_l2(a, bb[i], acc[i]);
            a += 1e-7f;
        }
        float r = 0; for (int i = 0; i < 8; ++i) r += __uint_as_float((unsigned)acc[i]) + __uint_as_float((unsigned)(acc[i] >> 32));
        out[blockIdx.x * blockDim.x + threadIdx.x] = r;
    } else if (MODE == 2) {  // scalar FFMA only: 16 chains
        float acc[16];
        for (int i = 0; i < 16; ++i) acc[i] = i;
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int i = 0; i < 16; ++i) acc[i] = __fmaf_rn(a, acc[i], b0);
        }
        float r = 0; for (int i = 0; i < 16; ++i) r += acc[i];
        out[blockIdx.x * blockDim.x + threadIdx.x] = r;
    } else {  // packed FFMA2 only: 8 packed chains
        unsigned long long acc[8], aa, bb;
        asm("mov.b64 %0, {%1,%1};" : "=l"(aa) : "f"(a));
        asm("mov.b64 %0, {%1,%2};" : "=l"(bb) : "f"(b0), "f"(b1));
        for (int i = 0; i < 8; ++i) acc[i] = bb + i;
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int i = 0; i < 8; ++i) acc[i] = f2_fma(aa, acc[i], bb);
        }
        float r = 0; for (int i = 0; i < 8; ++i) r += __uint_as_float((unsigned)acc[i]);
        out[blockIdx.x * blockDim.x + threadIdx.x] = r;
    }
}
int main() {
    float* out; cudaMalloc(&out, 148 * 8 * 256 * sizeof(float));
    const int iters = 20000;
    const char* names[4] = {"scalar L2 (FADD+FFMA)", "packed L2 (FADD2+FFMA2)", "scalar FFMA", "packed FFMA2"};
    for (int mode = 0; mode < 4; ++mode) {
        for (int warps = 4; warps <= 32; warps *= 2) {
            cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
            auto launch = [&]() {
                if (mode == 0) k<0><<<148 * 2, warps * 16, 0>>>(out, iters, 1.f);
                if (mode == 1) k<1><<<148 * 2, warps * 16, 0>>>(out, iters, 1.f);
                if (mode == 2) k<2><<<148 * 2, warps * 16, 0>>>(out, iters, 1.f);
                if (mode == 3) k<3><<<148 * 2, warps * 16, 0>>>(out, iters, 1.f);
            };
            launch(); cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            // lane-ops: modes 0/1: 16 pairs x 2 ops per iter; 2/3: 16 fma per iter
            double ops = 148.0 * 2 * warps * 16 * (double)iters * (mode < 2 ? 32 : 16);
            printf("%-26s warps/SM %2d: %.3f ms  %.1f T lane-ops/s\n", names[mode], warps, ms, ops / ms / 1e9);
        }
    }
    return 0;
}
