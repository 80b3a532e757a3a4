// Microbenchmark: FFMA vs FFMA2 (packed fma.rn.f32x2, sm_100a) issue/throughput on the B200.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 ffma2.cu -o ffma2 && ./ffma2
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long f2(float2 v) { return *reinterpret_cast<unsigned long long*>(&v); }
__device__ __forceinline__ unsigned long long ffma2(unsigned long long a, unsigned long long b, unsigned long long c) {
    unsigned long long r;
    asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}

template <int MODE>
__global__ void k(float* out, int iters, float s) {
    float a[8];
    unsigned long long p[4];
    unsigned x = threadIdx.x;
    for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3f + i;
    for (int i = 0; i < 4; ++i) p[i] = f2(make_float2(a[2 * i], a[2 * i + 1]));
    const unsigned long long m = f2(make_float2(s, s)), c = f2(make_float2(0.5f, 0.5f));
    for (int it = 0; it < iters; ++it) {
        if (MODE == 0 || MODE == 2) {
#pragma unroll
            for (int i = 0; i < 8; ++i) a[i] = __fmaf_rn(a[i], s, 0.5f);
        } else {
#pragma unroll
            for (int i = 0; i < 4; ++i) p[i] = ffma2(p[i], m, c);
        }
        if (MODE >= 2) {  // 8 integer ops per iteration competing for issue
#pragma unroll
            for (int i = 0; i < 8; ++i) x = x * 3u + (unsigned)it;
        }
    }
    float r = 0.f;
    for (int i = 0; i < 8; ++i) r += a[i];
    for (int i = 0; i < 4; ++i) { float2 v = *reinterpret_cast<float2*>(&p[i]); r += v.x + v.y; }
    out[blockIdx.x * blockDim.x + threadIdx.x] = r + (float)x;
}

int main() {
    float* out;
    cudaMalloc(&out, 148 * 8 * 256 * sizeof(float));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int iters = 20000;
    const char* names[4] = {"FFMA x8", "FFMA2 x4", "FFMA x8 + 8 IMAD", "FFMA2 x4 + 8 IMAD"};
    for (int rep = 0; rep < 2; ++rep)
        for (int mode = 0; mode < 4; ++mode) {
            void (*fn)(float*, int, float) = mode == 0 ? k<0> : mode == 1 ? k<1> : mode == 2 ? k<2> : k<3>;
            fn<<<148 * 8, 256>>>(out, 10, 0.999f);
            cudaEventRecord(a);
            fn<<<148 * 8, 256>>>(out, iters, 0.999f);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            double flops = 2.0 * 8 * iters * 148.0 * 8 * 256;
            if (rep) printf("%-20s %8.3f ms  %7.1f TFLOP/s\n", names[mode], ms, flops / ms / 1e9);
        }
    return 0;
}
