// common.cuh — shared device code for the B200 ERP splatting path.
//
// Precision contract:
//  * All per-Gaussian geometry (K1 preprocess, K4b chain rule, the per-pair FP64 slow path) is
//    FP64 in the reference's operation order. Every TU is compiled with --fmad=false, so no
//    mul+add is ever contracted behind our back; FP32 hot loops use explicit __fmaf_rn.
//  * Per-pair blending is FP32 with a guard band: any pair whose FP32 decision (power < 0,
//    alpha < 1/255, T < 1e-4, the 0.99 clamp gate) is within the error bound of the threshold is
//    re-evaluated in FP64 exactly like proj/src/rasterizer.cpp:128-140.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace osb {

// ---------------------------------------------------------------- constants (rasterizer.hpp:18-23)
constexpr double kPi = 3.14159265358979323846;
constexpr double kAlphaMin = 1.0 / 255.0;
constexpr double kAlphaMax = 0.99;
constexpr double kTStop = 1e-4;
constexpr double kLowpass = 0.3;
constexpr double kNear = 0.01;
constexpr double kPole = 1e-4;  // camera.hpp:74
constexpr int kTile = 16;
constexpr int kTilePixels = kTile * kTile;
constexpr double kShC0 = 0.28209479177387814;  // scene.hpp:60

// T-stop guard (K3). Default: FP32 transmittance within a relative band of 2^-10
// of 1e-4 replays the pixel's prefix in FP64 (an empirical band: K3 frames equal the strict mode's
// on every parity scene). Strict mode (osplat_gpu_set_strict_guard): the band is a running bound e
// on the FP32 T's relative error against the FP64 loop — each contributing pair adds
// alpha / (1 - alpha) x (delta (1.001 + delta) + kAlphaErr), delta = K1's bound on the FP32 power
// error (alpha = o e^-power, so it is alpha's relative error), kAlphaErr the FP32 evaluation of
// o ex2(-power log2 e) (exponent rounding <= 5.6 x 2^-24, ex2.approx <= 2^-22, o and the product
// 2 x 2^-24) — plus kTStep per step for the roundings of 1 - alpha and T (1 - alpha); the decision is
// certain outside 1e-4 (1 +- (e + 2 e^2 + kTMargin)).
constexpr float kTBand = 1.0f / 1024.0f;
constexpr float kTLo = 1e-4f * (1.0f - kTBand);
constexpr float kTHi = 1e-4f * (1.0f + kTBand);
constexpr float kAlphaErr = 1.1e-6f;
constexpr float kTStep = 1.2e-7f;   // 2^-23
constexpr float kTMargin = 1e-6f;   // FP32 rounding of the threshold arithmetic
constexpr float kTPre = 2e-4f;      // T_next >= kTPre with e <= 0.25 is a certain continue

// Plane layout of the flat FP32 parameter / gradient / moment buffers (SoA, plane stride = stride):
//   0..2 position | 3 .. 3+3bc-1 SH (basis b, channel c -> 3 + 3b + c) | rotation w,x,y,z |
//   log-scale x,y,z | opacity logit.  planes = 11 + 3bc (59 at SH degree 3).
struct Planes {
    int bc;
    __host__ __device__ int sh(int b, int c) const { return 3 + 3 * b + c; }
    __host__ __device__ int rot(int k) const { return 3 + 3 * bc + k; }
    __host__ __device__ int lscale(int k) const { return 7 + 3 * bc + k; }
    __host__ __device__ int opacity() const { return 10 + 3 * bc; }
    __host__ __device__ int count() const { return 11 + 3 * bc; }
};

struct Pose {
    double R[9];  // row-major world->camera
    double t[3];
};

// Per-Gaussian blend record (FP32, 48 B) staged into shared memory by K3/K4a.
struct __align__(16) Splat32 {
    float ha, b, hc, o;          // 0.5*conic.a, conic.b, 0.5*conic.c, opacity
    float r, g, bl, pthr;        // SH colour, ln(255 * o)
    float dl, ext_x, ext_y, pad; // power guard band; half-extents (px) of the region where the
                                 // FP32 power can be <= pthr + dl (conservative, for culling);
                                 // pad = bits of "pre-clamp colour < 0" per channel (for K4b)
};

// ---------------------------------------------------------------- FP64 helpers (vecmath.hpp)
__device__ __forceinline__ double dot3(const double* a, const double* b) {
    return a[0] * b[0] + a[1] * b[1] + a[2] * b[2];
}
__device__ __forceinline__ void m3v(const double* m, const double* v, double* o) {
    double r0 = m[0] * v[0] + m[1] * v[1] + m[2] * v[2];
    double r1 = m[3] * v[0] + m[4] * v[1] + m[5] * v[2];
    double r2 = m[6] * v[0] + m[7] * v[1] + m[8] * v[2];
    o[0] = r0; o[1] = r1; o[2] = r2;
}
__device__ __forceinline__ void m3tv(const double* m, const double* v, double* o) {
    double r0 = m[0] * v[0] + m[3] * v[1] + m[6] * v[2];
    double r1 = m[1] * v[0] + m[4] * v[1] + m[7] * v[2];
    double r2 = m[2] * v[0] + m[5] * v[1] + m[8] * v[2];
    o[0] = r0; o[1] = r1; o[2] = r2;
}
// (2x3) x (3x3), s accumulated from 0.0 in k order.
__device__ __forceinline__ void m23_mul(const double* a, const double* r, double* o) {
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            double s = 0.0;
#pragma unroll
            for (int k = 0; k < 3; ++k) s += a[i * 3 + k] * r[k * 3 + j];
            o[i * 3 + j] = s;
        }
}
__device__ __forceinline__ void quat_rot(const double* q, double* r) {
    double w = q[0], x = q[1], y = q[2], z = q[3];
    r[0] = 1.0 - 2.0 * (y * y + z * z);
    r[1] = 2.0 * (x * y - w * z);
    r[2] = 2.0 * (x * z + w * y);
    r[3] = 2.0 * (x * y + w * z);
    r[4] = 1.0 - 2.0 * (x * x + z * z);
    r[5] = 2.0 * (y * z - w * x);
    r[6] = 2.0 * (x * z - w * y);
    r[7] = 2.0 * (y * z + w * x);
    r[8] = 1.0 - 2.0 * (x * x + y * y);
}
__device__ __forceinline__ double qnorm(const double* q) {
    return sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
}
__device__ __forceinline__ void qnormalize(const double* q, double* o) {
    double n = qnorm(q);
    o[0] = q[0] / n; o[1] = q[1] / n; o[2] = q[2] / n; o[3] = q[3] / n;
}
// Sigma = R diag(s^2) R^T from an already normalised quaternion (K4b: normalised once, by a
// reciprocal, for both Sigma and the rotation gradient).
__device__ __forceinline__ void covariance3d_unit(const double* qu, const double* s, double* sig);
// Sigma = R diag(s^2) R^T (scene.cpp:94-102), returned as the mirrored symmetric 3x3.
__device__ __forceinline__ void covariance3d(const double* q, const double* s, double* sig) {
    double qu[4];
    qnormalize(q, qu);
    covariance3d_unit(qu, s, sig);
}
__device__ __forceinline__ void covariance3d_unit(const double* qu, const double* s, double* sig) {
    double r[9];
    quat_rot(qu, r);
    double s2[3] = {s[0] * s[0], s[1] * s[1], s[2] * s[2]};
    double f[9];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            double acc = 0.0;
#pragma unroll
            for (int k = 0; k < 3; ++k) acc += r[i * 3 + k] * s2[k] * r[j * 3 + k];
            f[i * 3 + j] = acc;
        }
    sig[0] = f[0]; sig[1] = f[1]; sig[2] = f[2];
    sig[3] = f[1]; sig[4] = f[4]; sig[5] = f[5];
    sig[6] = f[2]; sig[7] = f[5]; sig[8] = f[8];
}

// Real SH basis up to degree 3, 3DGS signs (scene.cpp:45-67).
__device__ __forceinline__ void sh_basis(const double* d, int degree, double* b) {
    constexpr double C1 = 0.4886025119029199;
    constexpr double C20 = 1.0925484305920792, C21 = -1.0925484305920792, C22 = 0.31539156525252005,
                     C23 = -1.0925484305920792, C24 = 0.5462742152960396;
    constexpr double C30 = -0.5900435899266435, C31 = 2.890611442640554, C32 = -0.4570457994644658,
                     C33 = 0.3731763325901154, C34 = -0.4570457994644658, C35 = 1.445305721320277,
                     C36 = -0.5900435899266435;
    b[0] = kShC0;
    if (degree < 1) return;
    double x = d[0], y = d[1], z = d[2];
    b[1] = -C1 * y;
    b[2] = C1 * z;
    b[3] = -C1 * x;
    if (degree < 2) return;
    double xx = x * x, yy = y * y, zz = z * z;
    b[4] = C20 * x * y;
    b[5] = C21 * y * z;
    b[6] = C22 * (2.0 * zz - xx - yy);
    b[7] = C23 * x * z;
    b[8] = C24 * (xx - yy);
    if (degree < 3) return;
    b[9] = C30 * y * (3.0 * xx - yy);
    b[10] = C31 * x * y * z;
    b[11] = C32 * y * (4.0 * zz - xx - yy);
    b[12] = C33 * z * (2.0 * zz - 3.0 * xx - 3.0 * yy);
    b[13] = C34 * x * (4.0 * zz - xx - yy);
    b[14] = C35 * z * (xx - yy);
    b[15] = C36 * x * (xx - 3.0 * yy);
}

// ---------------------------------------------------------------- device bit helpers
__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm volatile("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}
__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(uint32_t* p, uint32_t v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// ---- TMA bulk staging (cp.async.bulk + mbarrier): K1 / K4b stage their CTA's parameter tile ----
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_wait_parity(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "MBAR_WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra MBAR_WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// Programmatic dependent launch (K2's chain of short kernels): a kernel launched with
// launch_pdl waits for its predecessor's completion and memory (griddepcontrol.wait) before reading
// anything the predecessor wrote, then lets its own successor be scheduled onto SMs as they free up
// (griddepcontrol.launch_dependents) — the successor's launch and ramp overlap this kernel's tail.
__device__ __forceinline__ void pdl_begin() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// std::remainder(x, w) (rasterizer.cpp:13 wrap_dx) for |x| < 1.5 w, where the quotient rounds to
// -1, 0 or +1 (a tie at |x| = w/2 rounds to the even 0) and x -/+ w is exact (Sterbenz). Centres
// lie in [0, W] and pixel centres in (0, W), so |x| < W always; anything else takes the libm path.
__device__ __forceinline__ double wrap_remainder(double x, double w) {
    const double h = 0.5 * w;
    if (!(fabs(x) < 1.5 * w)) return remainder(x, w);
    if (x > h) return x - w;
    if (x < -h) return x + w;
    return x;
}

// Exact FP64 evaluation of one (pixel, splat) pair — proj/src/rasterizer.cpp:128-134 and
// proj/src/gradients.cpp:125-132. Returns 0 when skipped; sx, sy are pixel centres.
__device__ __forceinline__ int pair_fp64(double px, double py, double ca, double cb, double cc,
                                         double o, double sx, double sy, double width, double* g_out,
                                         double* alpha_out) {
    double dx = wrap_remainder(px - sx, width);
    double dy = py - sy;
    double power = 0.5 * (ca * dx * dx + cc * dy * dy) + cb * dx * dy;
    if (power < 0.0) return 0;
    // Certain skips first: an FP32 estimate of alpha (relative error < 1e-4 here: the FP64->FP32
    // roundings of o and power plus ex2.approx) below 0.99/255 means the FP64 alpha is below
    // 1/255 too, so the (costly) FP64 exp is only evaluated for pairs that can contribute.
    if (static_cast<float>(o) * __expf(-static_cast<float>(power)) < 0.99f * static_cast<float>(kAlphaMin)) return 0;
    double g = exp(-power);
    double ab = o * g;
    double alpha = ab < kAlphaMax ? ab : kAlphaMax;
    if (alpha < kAlphaMin) return 0;
    *g_out = g;
    *alpha_out = alpha;
    return 1;
}

}  // namespace osb
