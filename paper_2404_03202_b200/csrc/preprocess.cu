// preprocess.cu — K1: per-Gaussian ERP preprocessing, one thread per Gaussian, FP64 geometry.
//
// Replaces project_gaussian + the tile-rect half of bin_to_tiles
// (proj/src/rasterizer.cpp:17-55, :65-78). Reads the SoA FP32 parameter planes once
// (coalesced: every plane access of a warp is one 128-B line), writes per-Gaussian records
// indexed by Gaussian id (no compaction: culled Gaussians get depth_key = ~0 and 0 tiles).
// HBM-bound: 44 + 12 bc bytes read per Gaussian + ~120 B written for visible ones.
#include "kernels.h"
#include "project.cuh"

namespace osb {

namespace {

// The record half of K1 shared with the projection import: tile rectangle (pole clamp, seam wrap),
// depth keys, FP64 guard copy and the FP32 blend record with its guard band and extents.
__device__ __forceinline__ void write_record(int gid, const double* p, const double* cov, const double* conic,
                                             double o, double t_r, const double* col, uint32_t neg_bits,
                                             double radius, int W, int H, const PreprocessOut& out) {
    const double a = cov[0], b = cov[1], c = cov[2];
    const double mid = 0.5 * (a + c);
    const double dd2 = 0.25 * (a - c) * (a - c) + b * b;
    const double dd = sqrt(dd2 > 0.0 ? dd2 : 0.0);
    const double lmax = mid + dd;

    // Tile rectangle with pole clamp and seam wrap (rasterizer.cpp:65-78).
    const int tiles_x = (W + kTile - 1) / kTile;
    const int tiles_y = (H + kTile - 1) / kTile;
    int ty0 = static_cast<int>(floor((p[1] - radius) / kTile));
    int ty1 = static_cast<int>(floor((p[1] + radius) / kTile));
    ty0 = ty0 > 0 ? ty0 : 0;
    ty1 = ty1 < tiles_y - 1 ? ty1 : tiles_y - 1;
    int tx0 = static_cast<int>(floor((p[0] - radius) / kTile));
    int tx1 = static_cast<int>(floor((p[0] + radius) / kTile));
    if (tx1 - tx0 + 1 >= tiles_x) {
        tx0 = 0;
        tx1 = tiles_x - 1;
    }
    const uint32_t touched = ty0 > ty1 ? 0u : static_cast<uint32_t>((ty1 - ty0 + 1) * (tx1 - tx0 + 1));

    // FP32 blend record and the guard band on `power`. Pairs with power within
    // delta of pthr = ln(255 o) or of 0 are resolved by the FP64 path in K3/K4a.
    const double qa = conic[0], qb = conic[1], qc = conic[2];
    // ln(255 o) only places the FP32 classifier's band, never a decision itself: FP32 logf (<= 1 ulp,
    // < 5e-7 absolute below ln 255 + the argument's rounding 6e-8) instead of the FP64 log, its error
    // added to the band below (+1e-6)
    const double pthr = static_cast<double>(logf(static_cast<float>(255.0 * o)));
    const double lmin = mid - dd;
    const double lam_q_max = 1.0 / (lmin > 1e-300 ? lmin : 1e-300);
    const double P_ = (pthr > 0.0 ? pthr : 0.0) + 1.0;
    const double dmax = sqrt(2.0 * P_ * lmax);
    const double tmax = 0.5 * (fabs(qa) + fabs(qb) + fabs(qc)) * dmax * dmax;
    double delta = 0x1p-20 * (tmax + lam_q_max * dmax * (dmax + 16.0)) + 0x1p-21 * fabs(pthr) + 2e-6;
    if (!(delta < 1e30)) delta = 1e30;

    out.depth_key[gid] = static_cast<uint64_t>(__double_as_longlong(t_r));
    // FP32 bits of t_r (monotone for positive values) and the frame's visible range of them (the
    // depth-rank sort keys are these bits relative to the minimum, shifted into 24 bits)
    const uint32_t dbits = __float_as_uint(__double2float_rn(t_r));
    out.depth_key32[gid] = dbits;
    const uint32_t act = __activemask();
    const uint32_t wmin = __reduce_min_sync(act, dbits), wmax = __reduce_max_sync(act, dbits);
    if ((threadIdx.x & 31) == __ffs(act) - 1) {
        atomicMin(out.depth_range, wmin);
        atomicMin(out.depth_range + 1, ~wmax);
    }
    out.touched[gid] = touched;
    out.radius[gid] = static_cast<float>(radius);
    out.rect[gid] = make_int4(tx0, tx1, ty0, ty1);
    out.pxy[gid] = make_double2(p[0], p[1]);
    out.conic_o[gid] = make_double4(qa, qb, qc, o);
    Splat32 s;
    s.ha = static_cast<float>(0.5 * qa);
    s.b = static_cast<float>(qb);
    s.hc = static_cast<float>(0.5 * qc);
    s.o = static_cast<float>(o);
    s.r = static_cast<float>(col[0]);
    s.g = static_cast<float>(col[1]);
    s.bl = static_cast<float>(col[2]);
    s.pthr = static_cast<float>(pthr);
    s.dl = static_cast<float>(delta);
    // Bounding box of {d : 0.5 d^T Q d <= P} is |dx| <= sqrt(2 P cov_a), |dy| <= sqrt(2 P cov_c)
    // (cov = Q^-1). With P = pthr + 3 delta (+ slack) every pixel outside has FP32 power
    // > pthr + delta, i.e. a certain skip, so culling by these extents preserves every decision.
    // (>= 0: only an imported record can have o < 1/255, and it never passes the alpha test)
    const double Pext = fmax((pthr + 3.0 * delta) * (1.0 + 1e-4) + 1e-3, 0.0);
    // (FP32 sqrt of the FP32-rounded argument: relative error ~1e-7, inside the 1e-5 slack)
    const double ex = static_cast<double>(sqrtf(static_cast<float>(2.0 * Pext * (a > 0.0 ? a : 0.0)))) * (1.0 + 1e-5) + 0.02;
    const double ey = static_cast<double>(sqrtf(static_cast<float>(2.0 * Pext * (c > 0.0 ? c : 0.0)))) * (1.0 + 1e-5) + 0.02;
    s.ext_x = ex < 1e30 ? static_cast<float>(ex) : 1e30f;
    s.ext_y = ey < 1e30 ? static_cast<float>(ey) : 1e30f;
    s.pad = __uint_as_float(neg_bits);  // K4b's colour-clamp gate
    out.splat[gid] = s;
}

#ifndef OSB_K1_LAZY_BAND
#define OSB_K1_LAZY_BAND 1e-9  // (A/B: a huge band re-sums every channel in the backward's order)
#endif
constexpr int kPreThreads = 128;  // Gaussians per CTA = one 512-B row per parameter plane

// 0.5 + sum_k c_k b_k(dir) in the backward's order (gradients.cpp:197-198) for one colour channel;
// coef points at basis 0's coefficient, basis k's is 3 * kPreThreads floats further (plane 3 + 3k + c).
// Out of line: only evaluated when the forward sum lies within 1e-9 of zero.
static __device__ __noinline__ double backward_order_sum(const double* dir, int degree, const float* coef) {
    double basis[16];
    sh_basis(dir, degree, basis);
    const int nb = (degree + 1) * (degree + 1);
    double r = 0.5;
    for (int k = 0; k < nb; ++k) r += static_cast<double>(coef[3 * kPreThreads * k]) * basis[k];
    return r;
}

// K1: one thread per Gaussian. The CTA's parameter tile (the active planes x 128 Gaussians: 59 rows
// of 512 B at SH degree 3) is staged into shared memory by TMA bulk copies issued by one thread
// and completed on an mbarrier — every load of the tile in flight at once, no registers held —
// instead of 59 dependent-latency global loads per thread (the parameter loads were K1's
// dominant stall: 30 % of its samples).
template <int DEG>
// (80 registers, 6 CTAs / SM; capped at 72 / 64 registers it spills: render 0.832 -> 0.845 / 0.851 ms)
__global__ void __launch_bounds__(kPreThreads) k_preprocess(const float* __restrict__ P, int n, int stride, int bc,
                                                            Pose pose, int W, int H, PreprocessOut out,
                                                            K2Scratch zero) {
    constexpr int active_degree = DEG;  // compile-time: the SH loop unrolls into registers
    constexpr int nb = (active_degree + 1) * (active_degree + 1);
    constexpr int kRows = 3 + 3 * nb + 8;  // position | active SH | rotation, log-scale, opacity
    __shared__ __align__(128) float s_par[kRows][kPreThreads];
    __shared__ __align__(8) uint64_t s_bar;
    const Planes pl{bc};
    const int g0 = blockIdx.x * kPreThreads;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&s_bar)) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    pdl_begin();  // the parameters may come from the previous step's Adam
    if (threadIdx.x == 0) {
        // rows end at a 16-B multiple; the planes are padded to the stride (a multiple of 32), so
        // the copy never leaves the plane
        const uint32_t bytes = (static_cast<uint32_t>(min(kPreThreads, n - g0)) * 4u + 15u) & ~15u;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&s_bar)),
                     "r"(bytes * kRows)
                     : "memory");
#pragma unroll 1
        for (int r = 0; r < kRows; ++r) {
            // rows 0..2 + 3 nb: planes 0..; the last 8 rows: rotation / log-scale / opacity planes
            const int plane = r < 3 + 3 * nb ? r : r - (3 + 3 * nb) + pl.rot(0);
            bulk_g2s(&s_par[r][0], P + static_cast<size_t>(plane) * stride + g0, bytes, &s_bar);
        }
    }
    __syncthreads();  // the barrier's initialisation is visible to every thread
    if (zero.hist) {  // the frame's K2 scratch, cleared while the tile's copies are in flight
        const int gi = blockIdx.x * kPreThreads + threadIdx.x, step = gridDim.x * kPreThreads;
        for (int k = gi; k < zero.nhist; k += step) zero.hist[k] = 0u;
        for (int k = gi; k < zero.tiles; k += step) zero.ranges[k] = make_uint2(~0u, 0u);
        for (int k = gi; k < zero.nsums; k += step) zero.sums[k] = 0u;
        if (gi == 0) *zero.flag = 0u;
    }
    mbar_wait_parity(&s_bar, 0);
    const int gid = g0 + threadIdx.x;
    if (gid >= n) return;
    const int t = threadIdx.x;
    auto ld = [&](int plane) {
        return s_par[plane < 3 + 3 * nb ? plane : plane - pl.rot(0) + 3 + 3 * nb][t];
    };
    Proj64 pr;
    if (!project64(ld, pl, pose, W, H, pr)) {
        out.depth_key[gid] = ~0ull;
        out.depth_key32[gid] = 0xFFFFFFFFu;
        out.touched[gid] = 0;
        out.radius[gid] = -1.0f;
        return;
    }

    // eval_sh (scene.cpp:104-112): colour = max(0, sum c_i b_i + 0.5)
    double dir[3];
    view_dir(pose, pr.t, pr.t_r, dir);
    double basis[16];
    sh_basis(dir, active_degree, basis);
    double col[3] = {0.0, 0.0, 0.0};
    float cmax = 0.0f;  // largest |coefficient| (FP32, one register: K1 is bound by its FP64 pipe)
#pragma unroll
    for (int k = 0; k < nb; ++k) {
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const float coef = s_par[pl.sh(k, c)][t];
            col[c] += static_cast<double>(coef) * basis[k];
            cmax = fmaxf(cmax, fabsf(coef));
        }
    }
    col[0] += 0.5; col[1] += 0.5; col[2] += 0.5;
    // K4b's colour-clamp gate: the sign of the backward's pre-clamp sum, 0.5 + terms in basis order
    // (gradients.cpp:197-198). The two orders differ by rounding only: at most 17 roundings of partial
    // sums bounded by S = 0.5 + sum |c_k b_k| <= 0.5 + 48 max|c_k| (|b_k| <= 3 on the unit sphere), i.e.
    // < 2e-15 S. So the sign is re-summed in the backward's order (out of line) only when the forward
    // sum lies within max(1e-9, 1e-14 S) of zero.
    uint32_t neg_bits = 0u;
    const double band = fmax(OSB_K1_LAZY_BAND, 1e-14 * (0.5 + 48.0 * static_cast<double>(cmax)));
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        bool neg = col[c] < 0.0;
        if (fabs(col[c]) < band) neg = backward_order_sum(dir, active_degree, &s_par[pl.sh(0, c)][t]) < 0.0;
        neg_bits |= neg ? (1u << c) : 0u;
    }
    col[0] = col[0] > 0.0 ? col[0] : 0.0;
    col[1] = col[1] > 0.0 ? col[1] : 0.0;
    col[2] = col[2] > 0.0 ? col[2] : 0.0;

    // radius = ceil(3 sqrt(lambda_max)) (rasterizer.cpp:46, vecmath.hpp:158-162)
    const double a = pr.cov[0], b = pr.cov[1], c = pr.cov[2];
    const double mid = 0.5 * (a + c);
    const double dd2 = 0.25 * (a - c) * (a - c) + b * b;
    const double dd = sqrt(dd2 > 0.0 ? dd2 : 0.0);
    const double lmax = mid + dd;
    const double radius = ceil(3.0 * sqrt(lmax));
    write_record(gid, pr.p, pr.cov, pr.conic, pr.o, pr.t_r, col, neg_bits, radius, W, H, out);
}


// Host-supplied SplatProjection records (bin_to_tiles / blend_forward on host projections,
// rasterizer.cpp:57-157): the same record half as K1, from FP64 planes instead of the parameters.
__global__ void __launch_bounds__(256) k_import(const double* __restrict__ in, int n, int W, int H,
                                                PreprocessOut out) {
    const int gid = blockIdx.x * blockDim.x + threadIdx.x;
    if (gid >= n) return;
    auto f = [&](int plane) { return in[static_cast<size_t>(plane) * n + gid]; };
    const double p[2] = {f(0), f(1)};
    const double cov[3] = {f(2), f(3), f(4)};
    const double conic[3] = {f(5), f(6), f(7)};
    const double col[3] = {f(10), f(11), f(12)};
    write_record(gid, p, cov, conic, f(13), f(9), col, 0u, f(8), W, H, out);
}

// cov and t of every Gaussian (zeros when culled) for the full SplatProjection records of a frame
// (osplat_frame_splats); the same project64 as K1, so bit-identical to what K1 used.
__global__ void __launch_bounds__(128) k_detail(const float* __restrict__ P, int n, int stride, int bc, Pose pose,
                                                int W, int H, double* __restrict__ out) {
    const int gid = blockIdx.x * blockDim.x + threadIdx.x;
    if (gid >= n) return;
    const Planes pl{bc};
    Proj64 pr;
    const bool vis = project64<false>(P, stride, pl, gid, pose, W, H, pr);
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        out[static_cast<size_t>(k) * n + gid] = vis ? pr.cov[k] : 0.0;
        out[static_cast<size_t>(3 + k) * n + gid] = vis ? pr.t[k] : 0.0;
    }
}

}  // namespace

void launch_preprocess(const float* params, int n, int stride, int bc, int active_degree, const Pose& pose,
                       int W, int H, const PreprocessOut& out, cudaStream_t s, const K2Scratch& zero) {
    if (n <= 0) return;
    const int blocks = (n + kPreThreads - 1) / kPreThreads;
    switch (active_degree) {
        case 0: launch_pdl(k_preprocess<0>, blocks, kPreThreads, s, params, n, stride, bc, pose, W, H, out, zero); break;
        case 1: launch_pdl(k_preprocess<1>, blocks, kPreThreads, s, params, n, stride, bc, pose, W, H, out, zero); break;
        case 2: launch_pdl(k_preprocess<2>, blocks, kPreThreads, s, params, n, stride, bc, pose, W, H, out, zero); break;
        default: launch_pdl(k_preprocess<3>, blocks, kPreThreads, s, params, n, stride, bc, pose, W, H, out, zero); break;
    }
    OSB_LAUNCHED(1);
}

void launch_import_projections(const double* planes, int n, int W, int H, const PreprocessOut& out, cudaStream_t s) {
    if (n <= 0) return;
    k_import<<<(n + 255) / 256, 256, 0, s>>>(planes, n, W, H, out);
    OSB_LAUNCHED(1);
}

void launch_projection_detail(const float* params, int n, int stride, int bc, const Pose& pose, int W, int H,
                              double* out, cudaStream_t s) {
    if (n <= 0) return;
    k_detail<<<(n + 127) / 128, 128, 0, s>>>(params, n, stride, bc, pose, W, H, out);
    OSB_LAUNCHED(1);
}

}  // namespace osb
