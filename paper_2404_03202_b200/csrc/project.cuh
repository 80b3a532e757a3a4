// project.cuh — FP64 per-Gaussian projection onto the ERP screen, shared by K1 (preprocess)
// and K4b (per-Gaussian backward) so both see bit-identical t, J, Sigma, cov2 and conic.
// Operation order follows proj/src/rasterizer.cpp:17-55 and proj/src/camera.cpp:21-107.
#pragma once

#include "common.cuh"

namespace osb {

struct Proj64 {
    double t[3];
    double t_r;
    double p[2];
    double cov[3];    // a, b, c (low-pass filtered)
    double conic[3];  // inverse
    double o;         // activated opacity
    double jac[6];    // J = dp/dt (2x3)
    double m23[6];    // J W
    double s[3];      // activated scales
    double s3[9];     // Sigma3
    double q[4];      // raw quaternion
};

__device__ __forceinline__ double load_param(const float* __restrict__ P, int stride, int plane, int gid) {
    return static_cast<double>(__ldg(P + static_cast<size_t>(plane) * stride + gid));
}

// world_to_camera (camera.cpp:21-23).
__device__ __forceinline__ void world_to_camera(const Pose& pose, const double* m, double* t, double* t_r) {
    m3v(pose.R, m, t);
    t[0] = t[0] + pose.t[0];
    t[1] = t[1] + pose.t[1];
    t[2] = t[2] + pose.t[2];
    *t_r = sqrt(t[0] * t[0] + t[1] * t[1] + t[2] * t[2]);
}

// jacobian_equirect, Eqs. 11-16 (camera.cpp:52-68). Pole already rejected by the caller.
__device__ __forceinline__ void jacobian_equirect(const double* t, double t_r, int W, int H, double* j) {
    double tx = t[0], ty = t[1], tz = t[2];
    double u = tx * tx + tz * tz;
    double rho = sqrt(u);
    double r2 = t_r * t_r;
    double wf = W / (2.0 * kPi);
    double hf = H / kPi;
    j[0] = wf * tz / u;
    j[1] = 0.0;
    j[2] = -wf * tx / u;
    j[3] = -hf * tx * ty / (r2 * rho);
    j[4] = hf * rho / r2;
    j[5] = -hf * tz * ty / (r2 * rho);
}

// jacobian_equirect_grad: g[(r*3+c)*3+k] = dJ_rc/dt_k (camera.cpp:70-107).
__device__ __forceinline__ void jacobian_equirect_grad(const double* t, double t_r, int W, int H, double* g) {
    double tx = t[0], ty = t[1], tz = t[2];
    double u = tx * tx + tz * tz;
    double rho = sqrt(u);
    double r2 = t_r * t_r;
    double u2 = u * u;
    double wf = W / (2.0 * kPi);
    double hf = H / kPi;
    g[0] = -2.0 * wf * tx * tz / u2; g[1] = 0.0; g[2] = wf * (tx * tx - tz * tz) / u2;
    g[3] = 0.0; g[4] = 0.0; g[5] = 0.0;
    g[6] = wf * (tx * tx - tz * tz) / u2; g[7] = 0.0; g[8] = 2.0 * wf * tx * tz / u2;
    double base = hf / (r2 * rho);
    g[9] = -base * ty * (1.0 - 2.0 * tx * tx / r2 - tx * tx / u);
    g[10] = -base * tx * (1.0 - 2.0 * ty * ty / r2);
    g[11] = base * tx * ty * tz * (2.0 / r2 + 1.0 / u);
    g[12] = base * tx * (1.0 - 2.0 * u / r2);
    g[13] = -2.0 * hf * rho * ty / (r2 * r2);
    g[14] = base * tz * (1.0 - 2.0 * u / r2);
    g[15] = base * tx * ty * tz * (2.0 / r2 + 1.0 / u);
    g[16] = -base * tz * (1.0 - 2.0 * ty * ty / r2);
    g[17] = -base * ty * (1.0 - 2.0 * tz * tz / r2 - tz * tz / u);
}

// K4b's J and dJ/dt together, with one reciprocal per denominator instead of ~20 FP64 divisions:
// within a few ulp of the two functions above (K4b only produces gradients, held to 1e-3 relative;
// K1 keeps the divisions, whose results feed exact tile decisions).
__device__ __forceinline__ void jacobian_equirect_and_grad_fast(const double* t, double t_r, int W, int H, double* j,
                                                                double* g) {
    const double tx = t[0], ty = t[1], tz = t[2];
    const double u = tx * tx + tz * tz;
    const double rho = sqrt(u);
    const double r2 = t_r * t_r;
    const double inv_u = 1.0 / u, inv_r2 = 1.0 / r2, inv_rho = 1.0 / rho;
    const double wf = W / (2.0 * kPi);
    const double hf = H / kPi;
    j[0] = wf * tz * inv_u;
    j[1] = 0.0;
    j[2] = -wf * tx * inv_u;
    const double base = hf * inv_r2 * inv_rho;  // hf / (r2 rho)
    j[3] = -base * tx * ty;
    j[4] = hf * rho * inv_r2;
    j[5] = -base * tz * ty;
    const double inv_u2 = inv_u * inv_u;
    g[0] = -2.0 * wf * tx * tz * inv_u2; g[1] = 0.0; g[2] = wf * (tx * tx - tz * tz) * inv_u2;
    g[3] = 0.0; g[4] = 0.0; g[5] = 0.0;
    g[6] = g[2]; g[7] = 0.0; g[8] = -g[0];
    const double a = 2.0 * inv_r2;
    g[9] = -base * ty * (1.0 - a * tx * tx - tx * tx * inv_u);
    g[10] = -base * tx * (1.0 - a * ty * ty);
    g[11] = base * tx * ty * tz * (a + inv_u);
    g[12] = base * tx * (1.0 - a * u);
    g[13] = -2.0 * hf * rho * ty * inv_r2 * inv_r2;
    g[14] = base * tz * (1.0 - a * u);
    g[15] = g[11];
    g[16] = -base * tz * (1.0 - a * ty * ty);
    g[17] = -base * ty * (1.0 - a * tz * tz - tz * tz * inv_u);
}

// project_gaussian (rasterizer.cpp:17-55) minus the SH colour. Returns false when culled
// (t_r < 0.01, pole-degenerate, opacity < 1/255).
// ld(plane) returns this Gaussian's FP32 parameter of that plane (global memory, or K1's shared-
// memory staging of its CTA's parameter tile).
template <bool kPixel = true, typename Ld>
__device__ __forceinline__ bool project64(Ld ld, const Planes& pl, const Pose& pose, int W, int H, Proj64& pr) {
    // all 11 geometry parameters are loaded first: independent loads in flight together instead of
    // each waiting behind the FP64 math that precedes its use
    float lsf[3], qf[4];
#pragma unroll
    for (int k = 0; k < 3; ++k) lsf[k] = ld(pl.lscale(k));
#pragma unroll
    for (int k = 0; k < 4; ++k) qf[k] = ld(pl.rot(k));
    const double logit = static_cast<double>(ld(pl.opacity()));
    double m[3] = {static_cast<double>(ld(0)), static_cast<double>(ld(1)), static_cast<double>(ld(2))};
    world_to_camera(pose, m, pr.t, &pr.t_r);
    const double* t = pr.t;
    if (pr.t_r < kNear) return false;
    double rho = sqrt(t[0] * t[0] + t[2] * t[2]);
    if (rho <= kPole * pr.t_r) return false;
    pr.o = 1.0 / (1.0 + exp(-logit));
    if (pr.o < kAlphaMin) return false;

    if (kPixel) {  // project_equirect (camera.cpp:25-39); the backward does not need p
        double lon = atan2(t[0], t[2]);
        if (lon >= kPi) lon -= 2.0 * kPi;
        double sine = t[1] / pr.t_r;
        sine = sine < -1.0 ? -1.0 : (sine > 1.0 ? 1.0 : sine);
        double lat = asin(sine);
        double sx = lon / kPi, sy = 2.0 * lat / kPi;
        pr.p[0] = (sx + 1.0) * W * 0.5;
        pr.p[1] = (sy + 1.0) * H * 0.5;
    }

    jacobian_equirect(t, pr.t_r, W, H, pr.jac);
    m23_mul(pr.jac, pose.R, pr.m23);
#pragma unroll
    for (int k = 0; k < 3; ++k) pr.s[k] = exp(static_cast<double>(lsf[k]));
#pragma unroll
    for (int k = 0; k < 4; ++k) pr.q[k] = static_cast<double>(qf[k]);
    covariance3d(pr.q, pr.s, pr.s3);
    double sm0[3], sm1[3];
    m3v(pr.s3, pr.m23, sm0);
    m3v(pr.s3, pr.m23 + 3, sm1);
    double a = dot3(pr.m23, sm0) + kLowpass;
    double b = dot3(pr.m23, sm1);
    double c = dot3(pr.m23 + 3, sm1) + kLowpass;
    pr.cov[0] = a; pr.cov[1] = b; pr.cov[2] = c;
    double det = a * c - b * b;
    pr.conic[0] = c / det;
    pr.conic[1] = -b / det;
    pr.conic[2] = a / det;
    return true;
}

template <bool kPixel = true>
__device__ __forceinline__ bool project64(const float* __restrict__ P, int stride, const Planes& pl, int gid,
                                          const Pose& pose, int W, int H, Proj64& pr) {
    return project64<kPixel>([&](int plane) { return __ldg(P + static_cast<size_t>(plane) * stride + gid); }, pl,
                             pose, W, H, pr);
}

// View direction W^T t / t_r (rasterizer.cpp:51).
__device__ __forceinline__ void view_dir(const Pose& pose, const double* t, double t_r, double* dir) {
    m3tv(pose.R, t, dir);
    double inv = 1.0 / t_r;
    dir[0] = dir[0] * inv;
    dir[1] = dir[1] * inv;
    dir[2] = dir[2] * inv;
}

}  // namespace osb
