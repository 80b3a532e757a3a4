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

__global__ void __launch_bounds__(256) k_preprocess(const float* __restrict__ P, int n, int stride, int bc,
                                                    int active_degree, Pose pose, int W, int H,
                                                    PreprocessOut out) {
    const int gid = blockIdx.x * blockDim.x + threadIdx.x;
    if (gid >= n) return;
    const Planes pl{bc};
    Proj64 pr;
    if (!project64(P, stride, pl, gid, pose, W, H, pr)) {
        out.depth_key[gid] = ~0ull;
        out.touched[gid] = 0;
        return;
    }

    // eval_sh (scene.cpp:104-112): colour = max(0, sum c_i b_i + 0.5)
    double dir[3];
    view_dir(pose, pr.t, pr.t_r, dir);
    double basis[16];
    sh_basis(dir, active_degree, basis);
    const int nb = (active_degree + 1) * (active_degree + 1);
    double col[3] = {0.0, 0.0, 0.0};
    for (int k = 0; k < nb; ++k) {
        col[0] += load_param(P, stride, pl.sh(k, 0), gid) * basis[k];
        col[1] += load_param(P, stride, pl.sh(k, 1), gid) * basis[k];
        col[2] += load_param(P, stride, pl.sh(k, 2), gid) * basis[k];
    }
    col[0] += 0.5; col[1] += 0.5; col[2] += 0.5;
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

    // Tile rectangle with pole clamp and seam wrap (rasterizer.cpp:65-78).
    const int tiles_x = (W + kTile - 1) / kTile;
    const int tiles_y = (H + kTile - 1) / kTile;
    int ty0 = static_cast<int>(floor((pr.p[1] - radius) / kTile));
    int ty1 = static_cast<int>(floor((pr.p[1] + radius) / kTile));
    ty0 = ty0 > 0 ? ty0 : 0;
    ty1 = ty1 < tiles_y - 1 ? ty1 : tiles_y - 1;
    int tx0 = static_cast<int>(floor((pr.p[0] - radius) / kTile));
    int tx1 = static_cast<int>(floor((pr.p[0] + radius) / kTile));
    if (tx1 - tx0 + 1 >= tiles_x) {
        tx0 = 0;
        tx1 = tiles_x - 1;
    }
    const uint32_t touched = ty0 > ty1 ? 0u : static_cast<uint32_t>((ty1 - ty0 + 1) * (tx1 - tx0 + 1));

    // FP32 blend record and the guard band on `power`. Pairs with power within
    // delta of pthr = ln(255 o) or of 0 are resolved by the FP64 path in K3/K4a.
    const double qa = pr.conic[0], qb = pr.conic[1], qc = pr.conic[2];
    const double pthr = log(255.0 * pr.o);
    const double lmin = mid - dd;
    const double lam_q_max = 1.0 / (lmin > 1e-300 ? lmin : 1e-300);
    const double P_ = (pthr > 0.0 ? pthr : 0.0) + 1.0;
    const double dmax = sqrt(2.0 * P_ * lmax);
    const double tmax = 0.5 * (fabs(qa) + fabs(qb) + fabs(qc)) * dmax * dmax;
    double delta = 0x1p-20 * (tmax + lam_q_max * dmax * (dmax + 16.0)) + 0x1p-21 * fabs(pthr) + 1e-6;
    if (!(delta < 1e30)) delta = 1e30;

    out.depth_key[gid] = static_cast<uint64_t>(__double_as_longlong(pr.t_r));
    out.touched[gid] = touched;
    out.rect[gid] = make_int4(tx0, tx1, ty0, ty1);
    out.pxy[gid] = make_double2(pr.p[0], pr.p[1]);
    out.conic_o[gid] = make_double4(qa, qb, qc, pr.o);
    Splat32 s;
    s.ha = static_cast<float>(0.5 * qa);
    s.b = static_cast<float>(qb);
    s.hc = static_cast<float>(0.5 * qc);
    s.o = static_cast<float>(pr.o);
    s.r = static_cast<float>(col[0]);
    s.g = static_cast<float>(col[1]);
    s.bl = static_cast<float>(col[2]);
    s.pthr = static_cast<float>(pthr);
    out.splat[gid] = s;
    out.delta[gid] = static_cast<float>(delta);
}

}  // namespace

void launch_preprocess(const float* params, int n, int stride, int bc, int active_degree, const Pose& pose,
                       int W, int H, const PreprocessOut& out, cudaStream_t s) {
    if (n <= 0) return;
    k_preprocess<<<(n + 255) / 256, 256, 0, s>>>(params, n, stride, bc, active_degree, pose, W, H, out);
    OSB_LAUNCHED(1);
}

}  // namespace osb
