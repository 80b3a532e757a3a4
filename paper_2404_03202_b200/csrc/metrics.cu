// osplat_metrics on the device: PSNR and SSIM of two H x W x 3 double images, in FP64 like the
// reference (metrics.cpp:17-79; capi.cpp:287-296). Not on the training hot path — the evaluation
// metric behind the reference C ABI — so the kernels are plain FP64 sweeps:
//   k_metric_rows: per channel, the horizontal 11-tap zero-padded pass of x, y, x^2, y^2, xy
//                  (conv_same's first loop, metrics.cpp:33-42) -> 5 planar FP64 maps;
//   k_metric_ssim: the vertical pass (metrics.cpp:43-52) of the 5 maps, the SSIM map
//                  (metrics.cpp:113-123) and its per-channel sum, one FP64 atomic per block;
//   k_metric_sq:   sum (a - b)^2 over all 3 H W values (psnr's MSE numerator, metrics.cpp:64-74).
#include <cmath>

#include "common.cuh"
#include "kernels.h"

namespace osb {
namespace {

constexpr int kHalf = 5;  // 11-tap window, sigma 1.5 (metrics.cpp:13-27)

struct Win64 {
    double w[2 * kHalf + 1];
};

__device__ double block_sum64(double v, double* red) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) red[warp] = v;
    __syncthreads();
    double t = 0.0;
    if (warp == 0) {
        t = lane < static_cast<int>(blockDim.x >> 5) ? red[lane] : 0.0;
        for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    }
    return t;
}

// maps: 5 planes per channel, plane (c * 5 + k) * W * H; k = x, y, xx, yy, xy
__global__ void __launch_bounds__(256) k_metric_rows(const double* __restrict__ a, const double* __restrict__ b,
                                                     int W, int H, Win64 win, double* __restrict__ maps) {
    const int x = blockIdx.x * 256 + threadIdx.x;
    const int y = blockIdx.y;
    const int c = blockIdx.z;
    if (x >= W) return;
    const size_t row = static_cast<size_t>(y) * W;
    const int k0 = max(-kHalf, -x), k1 = min(kHalf, W - 1 - x);
    double s[5] = {0, 0, 0, 0, 0};
    for (int k = k0; k <= k1; ++k) {
        const double wk = win.w[k + kHalf];
        const size_t i = (row + x + k) * 3 + c;
        const double xv = a[i], yv = b[i];
        s[0] += wk * xv;
        s[1] += wk * yv;
        s[2] += wk * (xv * xv);
        s[3] += wk * (yv * yv);
        s[4] += wk * (xv * yv);
    }
    const size_t plane = static_cast<size_t>(W) * H;
    for (int m = 0; m < 5; ++m) maps[(static_cast<size_t>(c) * 5 + m) * plane + row + x] = s[m];
}

__global__ void __launch_bounds__(256) k_metric_ssim(const double* __restrict__ maps, int W, int H, Win64 win,
                                                     double* __restrict__ channel_sums) {
    __shared__ double red[8];
    const int c = blockIdx.z;
    const size_t plane = static_cast<size_t>(W) * H;
    const double* m0 = maps + static_cast<size_t>(c) * 5 * plane;
    double local = 0.0;
    const int x = blockIdx.x * 256 + threadIdx.x;
    const int y = blockIdx.y;
    if (x < W) {
        const int k0 = max(-kHalf, -y), k1 = min(kHalf, H - 1 - y);
        double s[5] = {0, 0, 0, 0, 0};
        for (int k = k0; k <= k1; ++k) {
            const double wk = win.w[k + kHalf];
            const size_t i = static_cast<size_t>(y + k) * W + x;
            for (int m = 0; m < 5; ++m) s[m] += wk * m0[m * plane + i];
        }
        constexpr double C1 = 0.01 * 0.01, C2 = 0.03 * 0.03;
        const double mx = s[0], my = s[1];
        const double var_x = s[2] - mx * mx;
        const double var_y = s[3] - my * my;
        const double cov = s[4] - mx * my;
        const double a1 = 2.0 * mx * my + C1;
        const double a2 = 2.0 * cov + C2;
        const double b1 = mx * mx + my * my + C1;
        const double b2 = var_x + var_y + C2;
        local = (a1 * a2) / (b1 * b2);
    }
    const double t = block_sum64(local, red);
    if (threadIdx.x == 0) atomicAdd(channel_sums + c, t);
}

__global__ void __launch_bounds__(256) k_metric_sq(const double* __restrict__ a, const double* __restrict__ b, long n,
                                                   double* __restrict__ out) {
    __shared__ double red[8];
    double acc = 0.0;
    for (long i = blockIdx.x * 256L + threadIdx.x; i < n; i += static_cast<long>(gridDim.x) * 256L) {
        const double d = a[i] - b[i];
        acc += d * d;
    }
    const double t = block_sum64(acc, red);
    if (threadIdx.x == 0) atomicAdd(out, t);
}

// perspective_crop (eval.cpp:21-61): pinhole S x S view of an H x W x 3 panorama, 90 degree field
// of view, pitch about X then yaw about Y (cos / sin from the host, as the reference's libm gives
// them), the ray projected with project_equirect (camera.cpp:25-39) and sampled bilinearly with the
// seam wrapped horizontally and rows clamped.
__global__ void k_perspective_crop(const double* __restrict__ pano, int W, int H, int S, double cp, double sp,
                                   double cyw, double syw, double* __restrict__ out) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y;
    if (x >= S) return;
    const double f = S * 0.5, c = S * 0.5;
    const double dx = (x + 0.5 - c) / f, dy = (y + 0.5 - c) / f, dz = 1.0;
    const double px = dx, py = cp * dy - sp * dz, pz = sp * dy + cp * dz;
    const double tx = cyw * px + syw * pz, ty = py, tz = -syw * px + cyw * pz;
    const double tr = sqrt(tx * tx + ty * ty + tz * tz);
    double lon = atan2(tx, tz);
    if (lon >= kPi) lon -= 2.0 * kPi;
    double sine = ty / tr;
    sine = sine < -1.0 ? -1.0 : (sine > 1.0 ? 1.0 : sine);
    const double lat = asin(sine);
    const double sx = lon / kPi, sy = 2.0 * lat / kPi;
    const double gx = (sx + 1.0) * W * 0.5 - 0.5, gy = (sy + 1.0) * H * 0.5 - 0.5;
    const int x0 = static_cast<int>(floor(gx)), y0 = static_cast<int>(floor(gy));
    const double fx = gx - x0, fy = gy - y0;
    const int xa = ((x0 % W) + W) % W, xb = (((x0 + 1) % W) + W) % W;
    const int ya = min(max(y0, 0), H - 1), yb = min(max(y0 + 1, 0), H - 1);
    for (int ch = 0; ch < 3; ++ch) {
        const double v00 = pano[(static_cast<size_t>(ya) * W + xa) * 3 + ch];
        const double v10 = pano[(static_cast<size_t>(ya) * W + xb) * 3 + ch];
        const double v01 = pano[(static_cast<size_t>(yb) * W + xa) * 3 + ch];
        const double v11 = pano[(static_cast<size_t>(yb) * W + xb) * 3 + ch];
        out[(static_cast<size_t>(y) * S + x) * 3 + ch] =
            (1 - fy) * ((1 - fx) * v00 + fx * v10) + fy * ((1 - fx) * v01 + fx * v11);
    }
}

}  // namespace

void launch_perspective_crop(const double* pano, int W, int H, int S, double yaw, double pitch, double* out,
                             cudaStream_t s) {
    if (S <= 0) return;
    const dim3 grid((S + 127) / 128, S);
    k_perspective_crop<<<grid, 128, 0, s>>>(pano, W, H, S, std::cos(pitch), std::sin(pitch), std::cos(yaw),
                                            std::sin(yaw), out);
    OSB_LAUNCHED(1);
}

void launch_metrics_f64(const double* a, const double* b, int W, int H, double* maps, double* sums, cudaStream_t s) {
    Win64 win;
    double total = 0.0;
    for (int i = 0; i < 2 * kHalf + 1; ++i) {
        const double d = i - kHalf;
        win.w[i] = std::exp(-d * d / (2.0 * 1.5 * 1.5));
        total += win.w[i];
    }
    for (int i = 0; i < 2 * kHalf + 1; ++i) win.w[i] /= total;
    OSB_CUDA_CHECK(cudaMemsetAsync(sums, 0, 4 * sizeof(double), s));
    const dim3 grid((W + 255) / 256, H, 3);
    k_metric_rows<<<grid, 256, 0, s>>>(a, b, W, H, win, maps);
    OSB_LAUNCHED(1);
    k_metric_ssim<<<grid, 256, 0, s>>>(maps, W, H, win, sums + 1);
    OSB_LAUNCHED(1);
    const long n = 3L * W * H;
    long blocks = (n + 255) / 256;
    if (blocks > 148 * 8) blocks = 148 * 8;
    k_metric_sq<<<static_cast<int>(blocks), 256, 0, s>>>(a, b, n, sums);
    OSB_LAUNCHED(1);
}

}  // namespace osb
