// adam.cu — K5: fused Adam over every parameter plane (proj/src/trainer.cpp:128-178).
//
// Adam: one launch over the flat planes x stride FP32 buffers (p, g, m, v) — or the element range
// [begin, begin + count) of them (the shard of a data-parallel rank) — float4 per thread,
// per-plane learning rate from the kernel argument table (position / SH DC / SH rest / rotation /
// log-scale / opacity groups), host-computed bias corrections (one global step, like the
// reference's AdamState::step). Optionally zeroes the gradient it consumed (saves the separate
// memset before the next backward). HBM-bound: 28 B (32 B with zeroing) per element.
#include "kernels.h"

namespace osb {

namespace {

__global__ void __launch_bounds__(256) k_adam(float4* __restrict__ p, float4* __restrict__ g, float4* __restrict__ m,
                                              float4* __restrict__ v, AdamArgs a) {
    pdl_begin();
    const long n4 = (a.begin + a.count) / 4;
    const float b1 = 0.9f, b2 = 0.999f;
    const float ob1 = 1.0f - 0.9f, ob2 = 1.0f - 0.999f;
    for (long i = a.begin / 4 + blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; i < n4;
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

}  // namespace

void launch_adam(float* params, float* grads, float* m, float* v, const AdamArgs& a, cudaStream_t s) {
    const long n4 = a.count / 4;
    if (n4 <= 0) return;
    long blocks = (n4 + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    launch_pdl(k_adam, static_cast<int>(blocks), 256, s, reinterpret_cast<float4*>(params),
               reinterpret_cast<float4*>(grads), reinterpret_cast<float4*>(m), reinterpret_cast<float4*>(v), a);
    OSB_LAUNCHED(1);
}

}  // namespace osb
