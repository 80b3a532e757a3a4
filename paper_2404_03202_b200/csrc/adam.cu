// adam.cu — K5: fused Adam over every parameter plane (proj/src/trainer.cpp:128-178), plus the
// L1 term of the photometric loss (trainer.cpp:25-71) used by the device-resident train step.
//
// Adam: one launch over the flat planes x stride FP32 buffers (p, g, m, v), float4 per thread,
// per-plane learning rate from the kernel argument table (position / SH DC / SH rest / rotation /
// log-scale / opacity groups), host-computed bias corrections (one global step, like the
// reference's AdamState::step). Optionally zeroes the gradient it consumed (saves the separate
// memset before the next backward). HBM-bound: 28 B (32 B with zeroing) per element.
#include "kernels.h"

namespace osb {

namespace {

__global__ void __launch_bounds__(256) k_adam(float4* __restrict__ p, float4* __restrict__ g, float4* __restrict__ m,
                                              float4* __restrict__ v, AdamArgs a) {
    const long n4 = static_cast<long>(a.planes) * a.stride / 4;
    const float b1 = 0.9f, b2 = 0.999f;
    const float ob1 = 1.0f - 0.9f, ob2 = 1.0f - 0.999f;
    for (long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; i < n4;
         i += static_cast<long>(gridDim.x) * blockDim.x) {
        const int plane = static_cast<int>((i * 4) / a.stride);
        const float lr = a.lr_plane[plane];
        float4 pp = p[i], gg = g[i], mm = m[i], vv = v[i];
        float* pv = &pp.x;
        float* gv = &gg.x;
        float* mv = &mm.x;
        float* vvv = &vv.x;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const float gr = gv[k];
            const float mk = b1 * mv[k] + ob1 * gr;
            const float vk = b2 * vvv[k] + ob2 * gr * gr;
            const float mhat = mk * a.inv_bias1;
            const float vhat = vk * a.inv_bias2;
            pv[k] = pv[k] - lr * mhat / (sqrtf(vhat) + 1e-15f);
            mv[k] = mk;
            vvv[k] = vk;
        }
        p[i] = pp;
        m[i] = mm;
        v[i] = vv;
        if (a.zero_grad) g[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
}

__global__ void __launch_bounds__(256) k_l1(const float* __restrict__ rgb, const float* __restrict__ gt, int W, int H,
                                            int keep_rows, double scale, float* __restrict__ d_image,
                                            double* __restrict__ abs_sum) {
    const long plane = static_cast<long>(W) * H;
    const long kept = static_cast<long>(W) * keep_rows;
    double local = 0.0;
    for (long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; i < 3 * plane;
         i += static_cast<long>(gridDim.x) * blockDim.x) {
        const long pix = i % plane;
        float grad = 0.0f;
        if (pix < kept) {
            const float d = rgb[i] - gt[i];
            local += fabs(static_cast<double>(d));
            grad = static_cast<float>(d > 0.0f ? scale : (d < 0.0f ? -scale : 0.0));
        }
        d_image[i] = grad;
    }
    // block reduction of the FP64 partial sums
    __shared__ double s[8];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) local += __shfl_down_sync(0xffffffffu, local, off);
    if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = local;
    __syncthreads();
    if (threadIdx.x < 32) {
        double t = threadIdx.x < blockDim.x / 32 ? s[threadIdx.x] : 0.0;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) t += __shfl_down_sync(0xffffffffu, t, off);
        if (threadIdx.x == 0) atomicAdd(abs_sum, t);
    }
}

}  // namespace

void launch_adam(float* params, float* grads, float* m, float* v, const AdamArgs& a, cudaStream_t s) {
    const long n4 = static_cast<long>(a.planes) * a.stride / 4;
    if (n4 <= 0) return;
    long blocks = (n4 + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    k_adam<<<static_cast<int>(blocks), 256, 0, s>>>(reinterpret_cast<float4*>(params), reinterpret_cast<float4*>(grads),
                                                   reinterpret_cast<float4*>(m), reinterpret_cast<float4*>(v), a);
    OSB_LAUNCHED(1);
}

void launch_l1_loss(const float* rgb, const float* gt, int W, int H, int keep_rows, double scale, float* d_image,
                    double* abs_sum, cudaStream_t s) {
    const long total = 3L * W * H;
    if (total <= 0) return;
    long blocks = (total + 255) / 256;
    if (blocks > 148 * 8) blocks = 148 * 8;
    k_l1<<<static_cast<int>(blocks), 256, 0, s>>>(rgb, gt, W, H, keep_rows, scale, d_image, abs_sum);
    OSB_LAUNCHED(1);
}

}  // namespace osb
