// kernels.h — host-side launchers for the sm_100a kernels (one TU per kernel family).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace osb {

// Kernel launches issued by this library (reported by bench.py as gpu_launches).
void count_launches(int k);
long long launches_total();

// ---- K1 preprocess (preprocess.cu) --------------------------------------------------------
struct PreprocessOut {
    uint64_t* depth_key;   // N: bit pattern of t_r (monotone), ~0 when culled
    uint32_t* depth_key32; // N: FP32 bit pattern of t_r (monotone), ~0 when culled
    uint32_t* depth_range; // {min bits, ~max bits} over visible Gaussians (both atomicMin, init ~0)
    uint32_t* touched;     // N: tile instances this Gaussian emits
    int4* rect;            // N: {tx0, tx1, ty0, ty1} (tx may wrap)
    double2* pxy;          // N: FP64 pixel centre
    double4* conic_o;      // N: FP64 conic a, b, c and opacity
    Splat32* splat;        // N: FP32 blend record (conic, opacity, colour, guard band, extents)
    float* radius;         // N: screen radius ceil(3 sqrt(lambda_max)), -1 when culled (DensifyStats)
};
// The frame's K2 scratch that must start at zero (launch_k2_zero's job); with zero.hist set, K1
// clears it on the way (one launch less in the K2 chain).
struct K2Scratch {
    uint32_t* hist = nullptr;  // both digit-total slots of the sort workspace
    int nhist = 0;
    uint32_t* flag = nullptr;  // long-run flag
    uint2* ranges = nullptr;   // tile ranges -> {~0u, 0}
    int tiles = 0;
    uint32_t* sums = nullptr;  // emission block sums
    int nsums = 0;
};
K2Scratch k2_scratch(void* sort_ws, uint32_t* long_run_flag, uint2* ranges, int tiles, void* scan_ws, int n);
void launch_preprocess(const float* params, int n, int stride, int bc, int active_degree, const Pose& pose,
                       int W, int H, const PreprocessOut& out, cudaStream_t s, const K2Scratch& zero = K2Scratch{});

// Host-supplied SplatProjection records (rasterizer.hpp:31-41) as kSplatPlanes FP64 planes of n:
// p.x, p.y, cov a, b, c, conic a, b, c, radius, depth, colour r, g, b, alpha_base. Writes the
// same per-record outputs as K1 (depth must be finite and >= 0).
constexpr int kSplatPlanes = 14;
void launch_import_projections(const double* planes, int n, int W, int H, const PreprocessOut& out, cudaStream_t s);

// cov (3 planes) then t (3 planes), n each, of every Gaussian; zeros when culled.
void launch_projection_detail(const float* params, int n, int stride, int bc, const Pose& pose, int W, int H,
                              double* out, cudaStream_t s);

// ---- K2 duplicate + sort (sort.cu) ----------------------------------------------------------
struct SortWorkspace;  // opaque, owned by the context
size_t radix_workspace_bytes(int n_max, int key_bytes);
// Stable LSD radix sort of (key, value) pairs on bits [0, bits). keys/vals are double-buffered:
// the result ends up in *_out when the function returns true, in *_in otherwise.
// first_keys: the first pass reads its keys from there instead of keys_in (left untouched);
// iota_vals: values are the element indices (vals_in is only a ping-pong buffer).
bool radix_sort_u64(uint64_t* keys_in, uint64_t* keys_out, uint32_t* vals_in, uint32_t* vals_out, int n,
                    int bits, void* ws, cudaStream_t s, const uint64_t* first_keys = nullptr, bool iota_vals = false,
                    bool hist_zeroed = false);
// n_dev: optional device-side count (the sort covers min(n, *n_dev) elements; grids sized by n).
// counts_ready (bits <= 16 only): the first pass's block counts and every pass's digit totals are
// already in ws (launch_scan_emit with tile_sort_ws = ws after tile_sort_prepare(ws)).
// tile_slot: the tile sort's digit totals live in the workspace's second slot, zeroed beforehand
// (K1 / launch_k2_zero, or tile_sort_prepare after a workspace reallocation).
// ranges (tile sort): the last pass writes the tile ranges instead of the sorted keys (ranges must
// start at {~0u, 0}: K1 / launch_k2_zero; empty tiles keep that and read as empty — K3 stores them back as
// {0, 0}); keys_in / keys_out then hold no sorted result.
bool radix_sort_u32(uint32_t* keys_in, uint32_t* keys_out, uint32_t* vals_in, uint32_t* vals_out, int n,
                    int bits, void* ws, cudaStream_t s, const uint32_t* n_dev = nullptr, bool counts_ready = false,
                    bool tile_slot = false, uint2* ranges = nullptr);
void tile_sort_prepare(void* ws, cudaStream_t s);
// Zero both digit-total slots of a sort workspace, the long-run flag and the tile ranges (one
// chained launch at the start of K2; hist_zeroed / tile_slot sorts then skip their own memsets).
// (+ the emission's block sums at the head of scan_ws, sized for n Gaussians)
void launch_k2_zero(void* sort_ws, uint32_t* long_run_flag, uint2* ranges, int tiles, void* scan_ws, int n,
                    cudaStream_t s);
// The fast depth rank: stable 3-pass sort of Gaussian ids 0..n-1 (no value input) by the 24-bit key
// (bits[i] - min) >> shift, the smallest shift that fits the visible range below 0xFFFFFF (culled ->
// 0xFFFFFF), computed on the fly by the first pass from K1's FP32 depth bits and their {min, ~max}
// range; the keys end up in ki/ko like radix_sort_u32.
bool radix_sort_depth24(const uint32_t* depth_bits, const uint32_t* range, uint32_t* ki, uint32_t* ko, uint32_t* vi,
                        uint32_t* vo, int n, void* ws, cudaStream_t s, bool hist_zeroed = false);
// Exclusive scan of touched[order[r]] fused with the emission of (tile, gid) instances in depth
// order; writes only instances below `capacity`; *total = M (device).
size_t scan_workspace_bytes(int n);
// The per-depth-rank emission records launch_scan_emit leaves in its workspace (valid for the
// frame's lifetime): first output (emission index of the rank's first instance), Gaussian id,
// packed tile rectangle {x0 & 0xFFFF | width << 16, y0}. Instance li of rank r (row-major over its
// rectangle, columns wrapped at the seam) has emission index rank_off[r] + li.
struct EmitArrays {
    const uint32_t* rank_off;
    const uint32_t* rank_gid;
    const int2* rank_rc;
};
EmitArrays scan_emit_arrays(void* ws, int n);
// cta_first: emit_ctas(capacity) + 1 words of scratch (first depth rank of every emission CTA).
long emit_ctas(uint32_t capacity);
// tile_sort_ws (optional): the emission also writes the tile sort's first upsweep into that
// radix_sort_u32 workspace (zeroed digit totals first: tile_sort_prepare), sized for `capacity`.
// depth_keys24 (fast depth rank): its sorted 24-bit keys — runs of equal keys are put in exact
// (FP64 depth_key, id) order on the way (a run longer than 64 raises *long_run_flag: redo the depth
// rank with the full 64-bit sort). The block sums in ws start at zero (K1 / launch_k2_zero; after a
// counting pass: scan_sums_reset).
void launch_scan_emit(const uint32_t* touched, const uint32_t* order, const int4* rect, int n, int tiles_x,
                      uint32_t* keys, uint32_t* vals, uint32_t capacity, uint32_t* total, void* ws,
                      uint32_t* cta_first, void* tile_sort_ws, cudaStream_t s, const uint32_t* depth_keys24 = nullptr,
                      const uint64_t* depth_key = nullptr, uint32_t* long_run_flag = nullptr);
void scan_sums_reset(void* ws, int n, cudaStream_t s);

// ---- K3 blend (blend.cu) --------------------------------------------------------------------
struct FrameBuffers {
    float* rgb;        // 3 planes of H*W
    float* T;          // H*W
    int* contrib;      // H*W
    int* last;         // H*W
    int* visited;      // H*W or nullptr: list entries evaluated per pixel (work counting only)
};
// Sums of per-pixel visited (forward pairs) and last_contrib (backward pairs) -> out[0], out[1].
void launch_work_count(const FrameBuffers& fb, int pixels, unsigned long long* out, cudaStream_t s);
// 3 FP32 planes -> interleaved H x W x 3 FP64 (the reference Image layout).
// pixels [p0, p1) of the planar FP32 image into H x W x 3 doubles (the whole image by default)
void launch_planar_to_hwc_f64(const float* rgb, size_t plane, double* out, cudaStream_t s, size_t p0 = 0,
                              size_t p1 = static_cast<size_t>(-1));
// strict: the T-stop guard band is the rigorous running error bound instead of the 2^-10 band
// (common.cuh); slower (more FP64 replays), decisions provably the FP64 reference's.
// ranges: read, and empty tiles left as {~0u, 0} by the fused tile sort are stored back as {0, 0}
// tile rows [row0, row1) only (row1 < 0: to the last row): a frame can be blended in bands so the
// host copy of one band overlaps the blending of the next (Engine::render_hwc).
void launch_blend(const uint32_t* inst_gid, uint2* ranges, const PreprocessOut& pp, int W, int H,
                  int tiles_x, int tiles_y, const float bg[3], const FrameBuffers& fb, cudaStream_t s,
                  bool strict = false, int row0 = 0, int row1 = -1);

// ---- K4 backward (backward.cu) --------------------------------------------------------------
// Deterministic K4a (optional mode, gradients.cpp:94-169's fixed-order reduction): per tile the 16
// quarters' partial sums of each entry are combined in a fixed order in shared memory and stored
// (no atomics) at the instance's emission index in inst_acc (9 floats each, zeroed by the caller);
// then one thread per depth rank sums its instances in emission order in FP64 into acc. Run to run
// bit-identical gradients. inv_rank: n u32 of scratch.
void launch_backward_pixels_det(const uint32_t* inst_gid, const uint2* ranges, const PreprocessOut& pp, int W,
                                int H, int tiles_x, int tiles_y, const float bg[3], const FrameBuffers& fb,
                                const float* d_image, const EmitArrays& em, int n, uint32_t* inv_rank,
                                float* inst_acc, float4* acc, cudaStream_t s);
void launch_backward_pixels(const uint32_t* inst_gid, const uint2* ranges, const PreprocessOut& pp, int W,
                            int H, int tiles_x, int tiles_y, const float bg[3], const FrameBuffers& fb,
                            const float* d_image, float4* acc, cudaStream_t s);
struct ScreenStats {
    float2* d_screen;       // N (latest view, overwritten for visible Gaussians)
    double* norm_sum;       // N (accumulated)
    int* hits;              // N (accumulated)
};
void launch_backward_gaussians(const float* params, int n, int stride, int bc, int active_degree,
                               const Pose& pose, int W, int H, const PreprocessOut& pp, const float4* acc,
                               float* grads, const ScreenStats& st, bool overwrite, cudaStream_t s);

// ---- K5 Adam + loss (adam.cu) ---------------------------------------------------------------
struct AdamArgs {
    float lr_plane[64];  // learning rate per plane (planes <= 59)
    float inv_bias1, inv_bias2;
    int planes, stride;
    int zero_grad;
    long begin, count;  // flat element range (multiples of 4)
};
void launch_adam(float* params, float* grads, float* m, float* v, const AdamArgs& a, cudaStream_t s);
// loss() of trainer.cpp:25-71 (loss.cu): (1 - lambda) L1 + lambda (1 - SSIM) over the top
// keep_rows rows of planar FP32 images; writes dL/dC planes (0 in masked rows) and accumulates
// sums[0] = sum |r - g| (FP64), sums[1..3] = per-channel SSIM map sums. g_planes: 9 * W * H floats
// of scratch (only used when lambda > 0).
void launch_loss(const float* rgb, const float* gt, int W, int H, int keep_rows, double lambda, float* d_image,
                 float* g_planes, double* sums, cudaStream_t s);

// sum over n of (a - b)^2 in FP64 -> *out (psnr's MSE numerator, metrics.cpp:64-74).
void launch_sq_err(const float* a, const float* b, long n, double* out, cudaStream_t s);

// osplat_metrics (metrics.cu): two H x W x 3 FP64 images -> sums[0] = sum (a - b)^2,
// sums[1..3] = per-channel sums of the SSIM map (metrics.cpp:17-79). maps: 15 W H doubles.
void launch_metrics_f64(const double* a, const double* b, int W, int H, double* maps, double* sums, cudaStream_t s);
// perspective_crop (eval.cpp:21-61) of an H x W x 3 FP64 panorama into an S x S x 3 pinhole view.
void launch_perspective_crop(const double* pano, int W, int H, int S, double yaw, double pitch, double* out,
                             cudaStream_t s);

// ---- densification (densify.cu) -------------------------------------------------------------
struct DensifyArgs {
    double grad_threshold;  // densify_grad_threshold
    double split_scale;     // scale_split_threshold * extent
    double log_split;       // ln(split_factor)
    double prune_opacity;
    double prune_scale;     // prune_scale_world * extent
    double prune_radius;    // prune_radius_px
    int radius_active;
};
void launch_observe(const float* radius, float* max_radius, int n, cudaStream_t s);
size_t densify_scan_workspace_bytes(long n);
void launch_exclusive_scan_u64(const unsigned long long* in, unsigned long long* out, long n, void* ws,
                               cudaStream_t s);  // ws[nblocks] = total
void launch_densify_mark(const float* P, int n, int stride, int bc, const double* norm_sum, const int* hits,
                         const DensifyArgs& a, unsigned long long* code, cudaStream_t s);
void launch_densify_sources(const unsigned long long* code, const unsigned long long* rank, int n, int* clone_src,
                            int* split_src, cudaStream_t s);
void launch_densify_keep(const float* P, int n, int stride, int bc, int nc, long total, const unsigned long long* code,
                         const int* clone_src, const int* split_src, const float* max_radius, const DensifyArgs& a,
                         unsigned long long* keep, cudaStream_t s);
void launch_densify_write(const float* P, const float* M, const float* V, int n, int stride, int bc, int nc, long total,
                          const unsigned long long* keep, const unsigned long long* dest, const int* clone_src,
                          const int* split_src, const double* normals, const DensifyArgs& a, float* P2, float* M2,
                          float* V2, int stride2, cudaStream_t s);
void launch_reset_opacity(float* opacity_plane, int n, double cap, cudaStream_t s);

}  // namespace osb

#define OSB_CUDA_CHECK(expr)                                                                    \
    do {                                                                                        \
        cudaError_t err__ = (expr);                                                             \
        if (err__ != cudaSuccess) throw ::osb::CudaError(err__, #expr, __FILE__, __LINE__);    \
    } while (0)

#define OSB_LAUNCHED(k)                          \
    do {                                         \
        OSB_CUDA_CHECK(cudaGetLastError());      \
        ::osb::count_launches(k);                \
    } while (0)

#include <stdexcept>
#include <string>
namespace osb {
struct CudaError : std::runtime_error {
    CudaError(cudaError_t e, const char* expr, const char* file, int line)
        : std::runtime_error(std::string("CUDA error ") + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) +
                             ") at " + file + ":" + std::to_string(line) + ": " + expr) {}
};
#ifndef OSB_PDL
#define OSB_PDL 1
#endif
// Launch with programmatic stream serialization allowed (the kernel must start with pdl_begin()).
template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, cudaStream_t s, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = 0;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = OSB_PDL;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    OSB_CUDA_CHECK(cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...));
}

}  // namespace osb
