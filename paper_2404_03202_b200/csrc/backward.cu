// backward.cu — K4a (per-pixel, reverse order) and K4b (per-Gaussian chain rule, FP64).
//
// K4a replaces backward() pass 1 + pass 2 (proj/src/gradients.cpp:96-169): same CTA/tile layout
// as K3, list walked back to front from each pixel's last_contrib, the 9 per-instance
// accumulators (d_colour 3, d_opacity, d_p 2, d_conic 3) reduced across the warp with shuffles and
// added with one vector red.global.add.v4.f32 per 4 values. Pair decisions are the forward's
// (pair.cuh); the 0.99 clamp gate (gradients.cpp:146) has its own FP64 guard.
//
// K4b replaces pass 3 (gradients.cpp:173-295): one thread per visible Gaussian, FP64 internals,
// re-derives t, J, Sigma and the conic with the same device code as K1 and accumulates the raw
// parameter gradients into the flat FP32 plane buffer (allreduce-able as one tensor).
#include "kernels.h"
#include "pair.cuh"
#include "project.cuh"

namespace osb {

namespace {

__device__ __forceinline__ void red_add_v4(float4* addr, float a, float b, float c, float d) {
    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(addr), "f"(a), "f"(b), "f"(c), "f"(d)
                 : "memory");
}

__global__ void __launch_bounds__(kStage) k_backward_pixels(const uint32_t* __restrict__ inst_gid,
                                                            const uint2* __restrict__ ranges, PreprocessOut pp,
                                                            int W, int H, int tiles_x, float bg0, float bg1,
                                                            float bg2, FrameBuffers fb,
                                                            const float* __restrict__ d_image,
                                                            float4* __restrict__ acc) {
    __shared__ StageSmem sm;
    __shared__ int s_max_last;
    const int tile = blockIdx.x;
    const int tx = tile % tiles_x, ty = tile / tiles_x;
    const int lx = threadIdx.x & 15, ly = threadIdx.x >> 4;
    const int px = tx * kTile + lx, py = ty * kTile + ly;
    const int lane = threadIdx.x & 31;
    const bool inside = px < W && py < H;
    const uint2 range = ranges[tile];
    const double width = W;
    const double xc = tx * kTile + 8.0, yc = ty * kTile + 8.0;
    const float lxo = lx - 7.5f, lyo = ly - 7.5f;
    const float halfW = 0.5f * W, fW = static_cast<float>(W);

    const size_t pix = static_cast<size_t>(py) * W + px;
    const size_t plane = static_cast<size_t>(W) * H;
    const int last = inside ? fb.last[pix] : 0;
    const float T_final = inside ? fb.T[pix] : 0.0f;
    const float dl0 = inside ? d_image[pix] : 0.0f;
    const float dl1 = inside ? d_image[plane + pix] : 0.0f;
    const float dl2 = inside ? d_image[2 * plane + pix] : 0.0f;
    const float bg_dot = bg0 * dl0 + bg1 * dl1 + bg2 * dl2;

    if (threadIdx.x == 0) s_max_last = 0;
    __syncthreads();
    if (last > 0) atomicMax(&s_max_last, last);
    __syncthreads();
    const int max_last = s_max_last;

    float T_acc = T_final;
    float s0 = 0.0f, s1 = 0.0f, s2 = 0.0f;     // suffix colour
    float lc0 = 0.0f, lc1 = 0.0f, lc2 = 0.0f;  // last colour
    float last_a = 0.0f;

    for (int hi = max_last; hi > 0; hi -= kStage) {
        const int lo = hi > kStage ? hi - kStage : 0;
        const int cnt = hi - lo;
        __syncthreads();
        if (threadIdx.x < cnt)
            stage_splat(sm, threadIdx.x, inst_gid[range.x + lo + threadIdx.x], pp.pxy, pp.splat, pp.delta, xc, yc,
                        width);
        __syncthreads();
        for (int j = cnt - 1; j >= 0; --j) {
            const int k = lo + j;
            float v0 = 0.f, v1 = 0.f, v2 = 0.f, v3 = 0.f, v4 = 0.f, v5 = 0.f, v6 = 0.f, v7 = 0.f, v8 = 0.f;
            bool has = false;
            if (k < last) {
                const float4 A = sm.a[j];
                const float4 B = sm.b[j];
                float dx, dy, power;
                bool unc;
                if (pair_power(A, B, lxo, lyo, halfW, fW, dx, dy, power, unc)) {
                    const float4 Cc = sm.c[j];
                    float alpha, g;
                    bool gate;
                    bool ok = true;
                    if (unc) {
                        Pair64 p;
                        ok = pair_slow(sm.gid[j], px, py, width, pp.pxy, pp.conic_o, &p);
                        alpha = static_cast<float>(p.alpha);
                        g = static_cast<float>(p.g);
                        gate = p.og < kAlphaMax;
                    } else {
                        g = ex2_approx(-power * kLog2e);
                        const float og = Cc.w * g;
                        alpha = fminf(0.99f, og);
                        const float band = 0.99f * (1.5f * fabsf(B.w) + 1e-6f);
                        if (fabsf(og - 0.99f) <= band) {
                            Pair64 p;
                            pair_slow(sm.gid[j], px, py, width, pp.pxy, pp.conic_o, &p);
                            gate = p.og < kAlphaMax;
                        } else {
                            gate = og < 0.99f;
                        }
                    }
                    if (ok) {
                        has = true;
                        const float one_m = 1.0f - alpha;
                        const float inv = __fdividef(1.0f, one_m);
                        T_acc = T_acc * inv;
                        const float wb = alpha * T_acc;
                        v0 = dl0 * wb;
                        v1 = dl1 * wb;
                        v2 = dl2 * wb;
                        const float oml = 1.0f - last_a;
                        s0 = __fmaf_rn(lc0, last_a, s0 * oml);
                        s1 = __fmaf_rn(lc1, last_a, s1 * oml);
                        s2 = __fmaf_rn(lc2, last_a, s2 * oml);
                        float d_alpha = (Cc.x - s0) * dl0;
                        d_alpha = __fmaf_rn(Cc.y - s1, dl1, d_alpha);
                        d_alpha = __fmaf_rn(Cc.z - s2, dl2, d_alpha);
                        d_alpha = d_alpha * T_acc - (T_final * inv) * bg_dot;
                        lc0 = Cc.x; lc1 = Cc.y; lc2 = Cc.z;
                        last_a = alpha;
                        if (gate) {
                            v3 = g * d_alpha;
                            const float d_power = -g * Cc.w * d_alpha;
                            const float qx = __fmaf_rn(2.0f * A.z, dx, B.x * dy);
                            const float qy = __fmaf_rn(B.x, dx, 2.0f * A.w * dy);
                            v4 = d_power * qx;
                            v5 = d_power * qy;
                            const float hp = 0.5f * d_power;
                            v6 = hp * dx * dx;
                            v7 = d_power * dx * dy;
                            v8 = hp * dy * dy;
                        }
                    }
                }
            }
            if (__any_sync(0xffffffffu, has)) {
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) {
                    v0 += __shfl_down_sync(0xffffffffu, v0, off);
                    v1 += __shfl_down_sync(0xffffffffu, v1, off);
                    v2 += __shfl_down_sync(0xffffffffu, v2, off);
                    v3 += __shfl_down_sync(0xffffffffu, v3, off);
                    v4 += __shfl_down_sync(0xffffffffu, v4, off);
                    v5 += __shfl_down_sync(0xffffffffu, v5, off);
                    v6 += __shfl_down_sync(0xffffffffu, v6, off);
                    v7 += __shfl_down_sync(0xffffffffu, v7, off);
                    v8 += __shfl_down_sync(0xffffffffu, v8, off);
                }
                if (lane == 0) {
                    float4* a = acc + 3 * static_cast<size_t>(sm.gid[j]);
                    red_add_v4(a, v0, v1, v2, v3);
                    red_add_v4(a + 1, v4, v5, v6, v7);
                    red_add_v4(a + 2, v8, 0.f, 0.f, 0.f);
                }
            }
        }
    }
}

// Real SH basis gradients w.r.t. the direction (scene.cpp:69-92); g is 16 x 3.
__device__ __forceinline__ void sh_basis_grad(const double* d, int degree, double* b, double* g) {
    constexpr double C1 = 0.4886025119029199;
    constexpr double C20 = 1.0925484305920792, C21 = -1.0925484305920792, C22 = 0.31539156525252005,
                     C23 = -1.0925484305920792, C24 = 0.5462742152960396;
    constexpr double C30 = -0.5900435899266435, C31 = 2.890611442640554, C32 = -0.4570457994644658,
                     C33 = 0.3731763325901154, C34 = -0.4570457994644658, C35 = 1.445305721320277,
                     C36 = -0.5900435899266435;
    sh_basis(d, degree, b);
    g[0] = 0.0; g[1] = 0.0; g[2] = 0.0;
    if (degree < 1) return;
    const double x = d[0], y = d[1], z = d[2];
    g[3] = 0.0; g[4] = -C1; g[5] = 0.0;
    g[6] = 0.0; g[7] = 0.0; g[8] = C1;
    g[9] = -C1; g[10] = 0.0; g[11] = 0.0;
    if (degree < 2) return;
    const double xx = x * x, yy = y * y, zz = z * z;
    g[12] = C20 * y; g[13] = C20 * x; g[14] = 0.0;
    g[15] = 0.0; g[16] = C21 * z; g[17] = C21 * y;
    g[18] = -2.0 * C22 * x; g[19] = -2.0 * C22 * y; g[20] = 4.0 * C22 * z;
    g[21] = C23 * z; g[22] = 0.0; g[23] = C23 * x;
    g[24] = 2.0 * C24 * x; g[25] = -2.0 * C24 * y; g[26] = 0.0;
    if (degree < 3) return;
    g[27] = C30 * 6.0 * x * y; g[28] = C30 * (3.0 * xx - 3.0 * yy); g[29] = 0.0;
    g[30] = C31 * y * z; g[31] = C31 * x * z; g[32] = C31 * x * y;
    g[33] = -2.0 * C32 * x * y; g[34] = C32 * (4.0 * zz - xx - 3.0 * yy); g[35] = 8.0 * C32 * y * z;
    g[36] = -6.0 * C33 * x * z; g[37] = -6.0 * C33 * y * z; g[38] = C33 * (6.0 * zz - 3.0 * xx - 3.0 * yy);
    g[39] = C34 * (4.0 * zz - 3.0 * xx - yy); g[40] = -2.0 * C34 * x * y; g[41] = 8.0 * C34 * x * z;
    g[42] = 2.0 * C35 * x * z; g[43] = -2.0 * C35 * y * z; g[44] = C35 * (xx - yy);
    g[45] = C36 * (3.0 * xx - 3.0 * yy); g[46] = -6.0 * C36 * x * y; g[47] = 0.0;
}

__device__ __forceinline__ void add_grad(float* __restrict__ G, int stride, int plane, int gid, double v) {
    float* p = G + static_cast<size_t>(plane) * stride + gid;
    *p = *p + static_cast<float>(v);
}

__global__ void __launch_bounds__(128) k_backward_gaussians(const float* __restrict__ P, int n, int stride, int bc,
                                                            int active_degree, Pose pose, int W, int H,
                                                            const uint64_t* __restrict__ depth_key,
                                                            const float4* __restrict__ acc, float* __restrict__ G,
                                                            ScreenStats st) {
    const int gid = blockIdx.x * blockDim.x + threadIdx.x;
    if (gid >= n || depth_key[gid] == ~0ull) return;
    const Planes pl{bc};
    Proj64 pr;
    project64(P, stride, pl, gid, pose, W, H, pr);  // visible by construction (same code as K1)

    const float4 a0 = acc[3 * static_cast<size_t>(gid)];
    const float4 a1 = acc[3 * static_cast<size_t>(gid) + 1];
    const float4 a2 = acc[3 * static_cast<size_t>(gid) + 2];
    const double d_color[3] = {a0.x, a0.y, a0.z};
    const double d_opacity = a0.w;
    const double d_p[2] = {a1.x, a1.y};
    const double dca_in = a1.z, dcb_in = a1.w, dcc_in = a2.x;

    // screen-space gradient and densification statistics (gradients.cpp:180-183)
    const double ds0 = d_p[0] * W * 0.5, ds1 = d_p[1] * H * 0.5;
    st.d_screen[gid] = make_float2(static_cast<float>(ds0), static_cast<float>(ds1));
    st.norm_sum[gid] += sqrt(ds0 * ds0 + ds1 * ds1);
    st.hits[gid] += 1;

    // opacity through the sigmoid (gradients.cpp:186-187)
    const double o = pr.o;
    add_grad(G, stride, pl.opacity(), gid, d_opacity * o * (1.0 - o));

    // colour: SH coefficients and the view-direction path (gradients.cpp:190-209)
    double dir[3];
    view_dir(pose, pr.t, pr.t_r, dir);
    double basis[16], dbasis[48];
    sh_basis_grad(dir, active_degree, basis, dbasis);
    const int active_n = (active_degree + 1) * (active_degree + 1);
    double raw[3] = {0.5, 0.5, 0.5};
    for (int i = 0; i < active_n; ++i)
        for (int c = 0; c < 3; ++c) raw[c] += load_param(P, stride, pl.sh(i, c), gid) * basis[i];
    double dlc[3];
    for (int c = 0; c < 3; ++c) dlc[c] = raw[c] < 0.0 ? 0.0 : d_color[c];
    double d_dir[3] = {0.0, 0.0, 0.0};
    for (int i = 0; i < active_n; ++i) {
        double co[3];
        for (int c = 0; c < 3; ++c) {
            co[c] = load_param(P, stride, pl.sh(i, c), gid);
            add_grad(G, stride, pl.sh(i, c), gid, dlc[c] * basis[i]);
        }
        const double cdot = co[0] * dlc[0] + co[1] * dlc[1] + co[2] * dlc[2];
        for (int c = 0; c < 3; ++c) d_dir[c] += dbasis[3 * i + c] * cdot;
    }
    const double dd = dot3(dir, d_dir);
    double d_m_sh[3];
    for (int c = 0; c < 3; ++c) d_m_sh[c] = (d_dir[c] - dir[c] * dd) * (1.0 / pr.t_r);

    // mean path: dL/dt = J^T dL/dp (gradients.cpp:212-213)
    const double* jac = pr.jac;
    double d_t[3] = {jac[0] * d_p[0] + jac[3] * d_p[1], jac[1] * d_p[0] + jac[4] * d_p[1],
                     jac[2] * d_p[0] + jac[5] * d_p[1]};

    // covariance path (gradients.cpp:216-254)
    const double qa = pr.conic[0], qb = pr.conic[1], qc = pr.conic[2];
    const double da = dca_in, db = 0.5 * dcb_in, dc = dcc_in;
    const double m00 = qa * da + qb * db, m01 = qa * db + qb * dc;
    const double m10 = qb * da + qc * db, m11 = qb * db + qc * dc;
    const double dva = -(m00 * qa + m01 * qb);
    const double dvb = -(m00 * qb + m01 * qc);
    const double dvc = -(m10 * qb + m11 * qc);
    const double* m0 = pr.m23;
    const double* m1 = pr.m23 + 3;
    double dsig[9];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c)
            dsig[r * 3 + c] = dva * m0[r] * m0[c] + dvb * (m0[r] * m1[c] + m1[r] * m0[c]) + dvc * m1[r] * m1[c];
    double sm0[3], sm1[3];
    m3v(pr.s3, m0, sm0);
    m3v(pr.s3, m1, sm1);
    double dm[6];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        dm[c] = (sm0[c] * dva + sm1[c] * dvb) * 2.0;
        dm[3 + c] = (sm0[c] * dvb + sm1[c] * dvc) * 2.0;
    }
    double Rt[9];
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) Rt[a * 3 + b] = pose.R[b * 3 + a];
    double djac[6];
    m23_mul(dm, Rt, djac);
    double jg[18];
    jacobian_equirect_grad(pr.t, pr.t_r, W, H, jg);
#pragma unroll
    for (int r = 0; r < 6; ++r) {
        const double dj = djac[r];
        d_t[0] += jg[3 * r + 0] * dj;
        d_t[1] += jg[3 * r + 1] * dj;
        d_t[2] += jg[3 * r + 2] * dj;
    }
    double dpos[3];
    m3tv(pose.R, d_t, dpos);
    for (int c = 0; c < 3; ++c) add_grad(G, stride, c, gid, dpos[c] + d_m_sh[c]);

    // Sigma3 -> quaternion (through normalisation) and log-scales (gradients.cpp:260-293)
    double qu[4], rot[9];
    qnormalize(pr.q, qu);
    quat_rot(qu, rot);
    const double* s = pr.s;
    double drot[9];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            double v = 0.0;
#pragma unroll
            for (int k = 0; k < 3; ++k) v += dsig[r * 3 + k] * rot[k * 3 + c];
            drot[r * 3 + c] = 2.0 * v * s[c] * s[c];
        }
    const double w = qu[0], x = qu[1], y = qu[2], z = qu[3];
    const double rg[4][9] = {{0, -2 * z, 2 * y, 2 * z, 0, -2 * x, -2 * y, 2 * x, 0},
                             {0, 2 * y, 2 * z, 2 * y, -4 * x, -2 * w, 2 * z, 2 * w, -4 * x},
                             {-4 * y, 2 * x, 2 * w, 2 * x, 0, 2 * z, -2 * w, 2 * z, -4 * y},
                             {-4 * z, -2 * w, 2 * x, 2 * w, -4 * z, 2 * y, 2 * x, 2 * y, 0}};
    double dqu[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        double v = 0.0;
#pragma unroll
        for (int i = 0; i < 9; ++i) v += drot[i] * rg[k][i];
        dqu[k] = v;
    }
    const double qn = qnorm(pr.q);
    const double qdot = qu[0] * dqu[0] + qu[1] * dqu[1] + qu[2] * dqu[2] + qu[3] * dqu[3];
    for (int k = 0; k < 4; ++k) add_grad(G, stride, pl.rot(k), gid, (dqu[k] - qu[k] * qdot) / qn);
    for (int k = 0; k < 3; ++k) {
        const double rk[3] = {rot[k], rot[3 + k], rot[6 + k]};
        double srk[3];
        m3v(dsig, rk, srk);
        const double rr = dot3(rk, srk);
        add_grad(G, stride, pl.lscale(k), gid, 2.0 * s[k] * rr * s[k]);
    }
}

}  // namespace

void launch_backward_pixels(const uint32_t* inst_gid, const uint2* ranges, const PreprocessOut& pp, int W, int H,
                            int tiles_x, int tiles_y, const float bg[3], const FrameBuffers& fb, const float* d_image,
                            float4* acc, cudaStream_t s) {
    const int tiles = tiles_x * tiles_y;
    if (tiles <= 0) return;
    k_backward_pixels<<<tiles, kStage, 0, s>>>(inst_gid, ranges, pp, W, H, tiles_x, bg[0], bg[1], bg[2], fb, d_image,
                                                acc);
    OSB_LAUNCHED(1);
}

void launch_backward_gaussians(const float* params, int n, int stride, int bc, int active_degree, const Pose& pose,
                               int W, int H, const uint64_t* depth_key, const float4* acc, float* grads,
                               const ScreenStats& st, cudaStream_t s) {
    if (n <= 0) return;
    k_backward_gaussians<<<(n + 127) / 128, 128, 0, s>>>(params, n, stride, bc, active_degree, pose, W, H, depth_key,
                                                          acc, grads, st);
    OSB_LAUNCHED(1);
}

}  // namespace osb
