// Microbenchmark: cost of a software grid-wide barrier in a persistent kernel (one CTA per SM
// slot, all co-resident) on B200 — the building block a single-kernel K2 would use instead of a
// chain of ~18 dependent launches. Prints us per barrier for several CTA counts, and the cost of
// an empty dependent-launch chain of the same length for comparison.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gridsync gridsync.cu && ./gridsync
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void grid_barrier(unsigned* count, volatile unsigned* gen, unsigned nblocks) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned g = *gen;
        __threadfence();
        if (atomicAdd(count, 1u) == nblocks - 1) {
            *count = 0;
            __threadfence();
            atomicAdd((unsigned*)gen, 1u);
        } else {
            while (*gen == g) {
            }
        }
        __threadfence();
    }
    __syncthreads();
}

__global__ void k_barriers(unsigned* count, unsigned* gen, int iters, float* sink) {
    float acc = threadIdx.x;
    for (int i = 0; i < iters; ++i) {
        acc = acc * 1.0001f + 1.0f;
        grid_barrier(count, gen, gridDim.x);
    }
    if (acc == -1.0f) sink[0] = acc;
}

__global__ void k_empty(float* sink) {
    if (threadIdx.x == 1023) sink[1] = 1.0f;
}

int main() {
    unsigned *count, *gen;
    float* sink;
    cudaMalloc(&count, 4);
    cudaMalloc(&gen, 4);
    cudaMalloc(&sink, 64);
    cudaMemset(count, 0, 4);
    cudaMemset(gen, 0, 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int per : {1, 2, 4}) {
        const int grid = sms * per, iters = 1000;
        k_barriers<<<grid, 256>>>(count, gen, 10, sink);
        cudaEventRecord(a);
        k_barriers<<<grid, 256>>>(count, gen, iters, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        printf("grid barrier: %d CTAs x 256 threads: %.3f us per barrier\n", grid, 1000.0f * ms / iters);
    }
    for (int blocks : {148, 600, 2000}) {
        const int n = 200;
        for (int i = 0; i < 10; ++i) k_empty<<<blocks, 256>>>(sink);
        cudaEventRecord(a);
        for (int i = 0; i < n; ++i) k_empty<<<blocks, 256>>>(sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        printf("empty kernel chain: %d blocks: %.3f us per launch\n", blocks, 1000.0f * ms / n);
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
