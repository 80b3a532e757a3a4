// densify.cu — gradient-driven densification on the device (proj/src/trainer.cpp:180-280).
//
// DensifyStats::observe (trainer.cpp:180-186): max screen radius per Gaussian over the trained
// views (K1 writes each frame's radius, -1 for culled).
//
// densify_and_prune (trainer.cpp:188-275) as a stream-compaction pipeline over the parameter
// planes: the reference's extended list [originals | clones | split children] is a virtual index
// space j in [0, n + nc + 2 ns); every j gets a keep flag, an exclusive scan of the flags gives the
// destination, and one gather kernel writes the surviving rows of the parameter and Adam planes
// into freshly allocated planes with the new stride. Decisions are taken in FP64 from the FP32
// parameters (exactly the values the reference would hold for an FP32-representable cloud):
//   clone/split:  mean |dL/ds| = norm_sum / hits >= threshold; split iff max(exp(log_scale)) >
//                 scale_split_threshold * extent (gradients.cpp:35-39, trainer.cpp:196-204)
//   children:     pos + R(q/|q|) (xi * s), xi ~ N(0, 1) drawn on the host from the reference's
//                 own std::mt19937_64 / std::normal_distribution stream (bit-identical draws),
//                 log_scale - ln(split_factor) (trainer.cpp:221-235)
//   prune:        split parents, sigmoid(logit) < prune_opacity, max scale > prune_scale_world *
//                 extent, max radius > prune_radius_px for originals after the first opacity reset
//                 (trainer.cpp:241-258).
// Scans: reduce-then-scan over 1024-element blocks (block sums -> one-block scan -> add), 64-bit
// values so clone and split counts travel packed in one pass.
#include "kernels.h"
#include "project.cuh"

namespace osb {

namespace {

constexpr int kScanBlock = 1024;  // elements per block (256 threads x 4)

__global__ void k_observe(const float* __restrict__ radius, float* __restrict__ max_radius, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float r = radius[i];
    if (r > max_radius[i]) max_radius[i] = r;
}

__device__ __forceinline__ double max3(double a, double b, double c) {  // std::max({a, b, c})
    double m = a;
    if (m < b) m = b;
    if (m < c) m = c;
    return m;
}

__device__ __forceinline__ double max_scale(const float* __restrict__ P, int stride, const Planes& pl, int i) {
    return max3(exp(load_param(P, stride, pl.lscale(0), i)), exp(load_param(P, stride, pl.lscale(1), i)),
                exp(load_param(P, stride, pl.lscale(2), i)));
}

// code[i] = 1 (clone) | 1 << 32 (split) packed for the scan; 0 otherwise.
__global__ void k_densify_mark(const float* __restrict__ P, int n, int stride, Planes pl,
                               const double* __restrict__ norm_sum, const int* __restrict__ hits, DensifyArgs a,
                               unsigned long long* __restrict__ code) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int h = hits[i];
    const double g = h == 0 ? 0.0 : norm_sum[i] / static_cast<double>(h);
    unsigned long long c = 0ull;
    if (!(g < a.grad_threshold)) c = max_scale(P, stride, pl, i) > a.split_scale ? (1ull << 32) : 1ull;
    code[i] = c;
}

// Block-level inclusive scan helper over 1024 elements (256 threads x 4 consecutive).
__device__ __forceinline__ unsigned long long block_exclusive(unsigned long long v, unsigned long long* sh,
                                                              unsigned long long* total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned long long x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) sh[warp] = x;
    __syncthreads();
    if (warp == 0) {
        unsigned long long w = lane < (blockDim.x >> 5) ? sh[lane] : 0ull;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        sh[lane] = w;
    }
    __syncthreads();
    const unsigned long long before = (warp > 0 ? sh[warp - 1] : 0ull) + x - v;
    if (total) *total = sh[(blockDim.x >> 5) - 1];
    __syncthreads();
    return before;
}

__global__ void __launch_bounds__(256) k_scan_reduce(const unsigned long long* __restrict__ in, int n,
                                                     unsigned long long* __restrict__ block_sums) {
    __shared__ unsigned long long sh[32];
    const long base = static_cast<long>(blockIdx.x) * kScanBlock + threadIdx.x * 4;
    unsigned long long s = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k)
        if (base + k < n) s += in[base + k];
    unsigned long long tot;
    block_exclusive(s, sh, &tot);
    if (threadIdx.x == 0) block_sums[blockIdx.x] = tot;
}

// One block: exclusive scan of the block sums in place; the grand total goes to block_sums[nb].
__global__ void __launch_bounds__(256) k_scan_sums(unsigned long long* __restrict__ block_sums, int nb) {
    __shared__ unsigned long long sh[32];
    unsigned long long carry = 0;
    for (int base = 0; base < nb; base += 256) {
        const int i = base + threadIdx.x;
        const unsigned long long v = i < nb ? block_sums[i] : 0ull;
        unsigned long long tot;
        const unsigned long long ex = block_exclusive(v, sh, &tot);
        if (i < nb) block_sums[i] = carry + ex;
        carry += tot;
    }
    if (threadIdx.x == 0) block_sums[nb] = carry;
}

__global__ void __launch_bounds__(256) k_scan_apply(const unsigned long long* __restrict__ in, int n,
                                                    const unsigned long long* __restrict__ block_sums,
                                                    unsigned long long* __restrict__ out) {
    __shared__ unsigned long long sh[32];
    const long base = static_cast<long>(blockIdx.x) * kScanBlock + threadIdx.x * 4;
    unsigned long long v[4], s = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        v[k] = base + k < n ? in[base + k] : 0ull;
        s += v[k];
    }
    unsigned long long run = block_sums[blockIdx.x] + block_exclusive(s, sh, nullptr);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        if (base + k < n) out[base + k] = run;
        run += v[k];
    }
}

__global__ void k_densify_sources(const unsigned long long* __restrict__ code, const unsigned long long* __restrict__ rank,
                                  int n, int* __restrict__ clone_src, int* __restrict__ split_src) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const unsigned long long c = code[i], r = rank[i];
    if (c & 0xffffffffull) clone_src[r & 0xffffffffull] = i;
    if (c >> 32) split_src[r >> 32] = i;
}

// Source row and kind of virtual entry j: kind 0 original, 1 clone, 2 split child (child index in
// *child: 2 * split rank + {0, 1}).
__device__ __forceinline__ int resolve(long j, int n, int nc, const int* __restrict__ clone_src,
                                       const int* __restrict__ split_src, int* src, int* child) {
    if (j < n) {
        *src = static_cast<int>(j);
        return 0;
    }
    if (j < static_cast<long>(n) + nc) {
        *src = clone_src[j - n];
        return 1;
    }
    const int c = static_cast<int>(j - n - nc);
    *child = c;
    *src = split_src[c >> 1];
    return 2;
}

__global__ void k_densify_keep(const float* __restrict__ P, int n, int stride, Planes pl, int nc, long total,
                               const unsigned long long* __restrict__ code, const int* __restrict__ clone_src,
                               const int* __restrict__ split_src, const float* __restrict__ max_radius, DensifyArgs a,
                               unsigned long long* __restrict__ keep) {
    const long j = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x;
    if (j >= total) return;
    int src = 0, child = 0;
    const int kind = resolve(j, n, nc, clone_src, split_src, &src, &child);
    unsigned long long k = 1ull;
    if (kind == 0 && (code[src] >> 32)) {
        k = 0ull;  // split parent
    } else {
        const double o = 1.0 / (1.0 + exp(-load_param(P, stride, pl.opacity(), src)));
        double s;
        if (kind == 2) {
            s = max3(exp(load_param(P, stride, pl.lscale(0), src) - a.log_split),
                     exp(load_param(P, stride, pl.lscale(1), src) - a.log_split),
                     exp(load_param(P, stride, pl.lscale(2), src) - a.log_split));
        } else {
            s = max_scale(P, stride, pl, src);
        }
        if (o < a.prune_opacity) k = 0ull;
        else if (s > a.prune_scale) k = 0ull;
        else if (a.radius_active && kind == 0 && static_cast<double>(max_radius[src]) > a.prune_radius) k = 0ull;
    }
    keep[j] = k;
}

// Gather the surviving rows into the new planes (stride2); Adam moments of new entries are zero.
__global__ void k_densify_write(const float* __restrict__ P, const float* __restrict__ M, const float* __restrict__ V,
                                int n, int stride, Planes pl, int nc, long total,
                                const unsigned long long* __restrict__ keep, const unsigned long long* __restrict__ dest,
                                const int* __restrict__ clone_src, const int* __restrict__ split_src,
                                const double* __restrict__ normals, DensifyArgs a, float* __restrict__ P2,
                                float* __restrict__ M2, float* __restrict__ V2, int stride2) {
    const long j = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x;
    if (j >= total || !keep[j]) return;
    const long d = static_cast<long>(dest[j]);
    int src = 0, child = 0;
    const int kind = resolve(j, n, nc, clone_src, split_src, &src, &child);
    const int planes = pl.count();
    for (int q = 0; q < planes; ++q) {
        P2[static_cast<size_t>(q) * stride2 + d] = P[static_cast<size_t>(q) * stride + src];
        M2[static_cast<size_t>(q) * stride2 + d] = kind == 0 ? M[static_cast<size_t>(q) * stride + src] : 0.0f;
        V2[static_cast<size_t>(q) * stride2 + d] = kind == 0 ? V[static_cast<size_t>(q) * stride + src] : 0.0f;
    }
    if (kind != 2) return;
    // split child (trainer.cpp:221-235): pos + R (xi * s), log_scale - ln(split_factor)
    double q4[4], qn[4], R[9], s[3], xi[3], dp[3];
    for (int k = 0; k < 4; ++k) q4[k] = load_param(P, stride, pl.rot(k), src);
    qnormalize(q4, qn);
    quat_rot(qn, R);
    for (int k = 0; k < 3; ++k) {
        const double ls = load_param(P, stride, pl.lscale(k), src);
        s[k] = exp(ls);
        xi[k] = normals[3 * static_cast<long>(child) + k] * s[k];
        P2[static_cast<size_t>(pl.lscale(k)) * stride2 + d] = static_cast<float>(ls - a.log_split);
    }
    m3v(R, xi, dp);
    for (int k = 0; k < 3; ++k)
        P2[static_cast<size_t>(k) * stride2 + d] = static_cast<float>(load_param(P, stride, k, src) + dp[k]);
}

// reset_opacity (trainer.cpp:277-280): logit = min(logit, cap) in FP64.
__global__ void k_reset_opacity(float* __restrict__ op, int n, double cap) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double l = static_cast<double>(op[i]);
    if (cap < l) op[i] = static_cast<float>(cap);
}

int blocks_for(long n, int per) { return static_cast<int>((n + per - 1) / per); }

}  // namespace

size_t densify_scan_workspace_bytes(long n) { return (static_cast<size_t>(blocks_for(n, kScanBlock)) + 1) * 8; }

void launch_observe(const float* radius, float* max_radius, int n, cudaStream_t s) {
    if (n <= 0) return;
    k_observe<<<blocks_for(n, 256), 256, 0, s>>>(radius, max_radius, n);
    OSB_LAUNCHED(1);
}

void launch_exclusive_scan_u64(const unsigned long long* in, unsigned long long* out, long n, void* ws,
                               cudaStream_t s) {
    if (n <= 0) return;
    const int nb = blocks_for(n, kScanBlock);
    unsigned long long* sums = static_cast<unsigned long long*>(ws);
    k_scan_reduce<<<nb, 256, 0, s>>>(in, static_cast<int>(n), sums);
    k_scan_sums<<<1, 256, 0, s>>>(sums, nb);
    k_scan_apply<<<nb, 256, 0, s>>>(in, static_cast<int>(n), sums, out);
    OSB_LAUNCHED(3);
}

void launch_densify_mark(const float* P, int n, int stride, int bc, const double* norm_sum, const int* hits,
                         const DensifyArgs& a, unsigned long long* code, cudaStream_t s) {
    if (n <= 0) return;
    k_densify_mark<<<blocks_for(n, 256), 256, 0, s>>>(P, n, stride, Planes{bc}, norm_sum, hits, a, code);
    OSB_LAUNCHED(1);
}

void launch_densify_sources(const unsigned long long* code, const unsigned long long* rank, int n, int* clone_src,
                            int* split_src, cudaStream_t s) {
    if (n <= 0) return;
    k_densify_sources<<<blocks_for(n, 256), 256, 0, s>>>(code, rank, n, clone_src, split_src);
    OSB_LAUNCHED(1);
}

void launch_densify_keep(const float* P, int n, int stride, int bc, int nc, long total, const unsigned long long* code,
                         const int* clone_src, const int* split_src, const float* max_radius, const DensifyArgs& a,
                         unsigned long long* keep, cudaStream_t s) {
    if (total <= 0) return;
    k_densify_keep<<<blocks_for(total, 256), 256, 0, s>>>(P, n, stride, Planes{bc}, nc, total, code, clone_src,
                                                          split_src, max_radius, a, keep);
    OSB_LAUNCHED(1);
}

void launch_densify_write(const float* P, const float* M, const float* V, int n, int stride, int bc, int nc, long total,
                          const unsigned long long* keep, const unsigned long long* dest, const int* clone_src,
                          const int* split_src, const double* normals, const DensifyArgs& a, float* P2, float* M2,
                          float* V2, int stride2, cudaStream_t s) {
    if (total <= 0) return;
    k_densify_write<<<blocks_for(total, 256), 256, 0, s>>>(P, M, V, n, stride, Planes{bc}, nc, total, keep, dest,
                                                           clone_src, split_src, normals, a, P2, M2, V2, stride2);
    OSB_LAUNCHED(1);
}

void launch_reset_opacity(float* opacity_plane, int n, double cap, cudaStream_t s) {
    if (n <= 0) return;
    k_reset_opacity<<<blocks_for(n, 256), 256, 0, s>>>(opacity_plane, n, cap);
    OSB_LAUNCHED(1);
}

}  // namespace osb
