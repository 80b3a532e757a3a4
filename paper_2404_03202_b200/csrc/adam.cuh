// adam.cuh — one element of adam_update (proj/src/trainer.cpp:128-139) in FP32, shared by K5
// (adam.cu) and the fused SH backward + Adam of the single-view step (backward.cu) so both make
// bit-identical updates: m = b1 m + (1 - b1) g, v = b2 v + (1 - b2) g^2,
// p -= lr (m / bias1) / (sqrt(v / bias2) + 1e-15).
#pragma once

namespace osb {

__device__ __forceinline__ void adam_elem(float& p, float& m, float& v, float gr, float lr, float inv_bias1,
                                          float inv_bias2) {
    const float b1 = 0.9f, b2 = 0.999f;
    const float ob1 = 1.0f - 0.9f, ob2 = 1.0f - 0.999f;
    const float mk = b1 * m + ob1 * gr;
    const float vk = b2 * v + ob2 * gr * gr;
    const float mhat = mk * inv_bias1;
    const float vhat = vk * inv_bias2;
    p = p - lr * mhat / (sqrtf(vhat) + 1e-15f);
    m = mk;
    v = vk;
}

}  // namespace osb
