// blend.cu — K3: per-tile front-to-back alpha blending (proj/src/rasterizer.cpp:100-157).
//
// One 256-thread CTA per 16x16 tile, one pixel per thread. The CTA stages the tile list 256
// entries at a time (each entry once, with a 16-quarter reach mask, pair.cuh), then each warp blends
// the staged entries in list order, each half-warp only those that can reach its 4x4 quarter; a
// warp stops as soon as its 32 pixels have terminated, the CTA when all have. FP32 fast path + FP64
// guard (pair.cuh): power/alpha decisions near a threshold and T near the 1e-4 stop are decided in
// FP64 exactly like the reference; a T decision inside the band replays the pixel's prefix in FP64
// (warp-cooperatively) and the pixel continues in FP64 ("exact mode").
#include <type_traits>

#include "kernels.h"
#include "pair.cuh"

namespace osb {

namespace {

#ifdef OSB_K3_STATS
// Instrumented build only (scripts/k4a_stats.py --k3): K3 lane-loop statistics per launch.
__device__ unsigned long long g_k3_stats[5];
#endif
#ifndef OSB_K3_PER
#define OSB_K3_PER 2  // entries staged per thread per round (512-entry rounds)
#endif
#ifndef OSB_K3_ELLIPSE
#define OSB_K3_ELLIPSE false  // K3 stages box masks (per-row ellipse intervals: measured slower in K3)
#endif
#ifndef OSB_K3_CTAS
#define OSB_K3_CTAS 4  // CTAs per SM (64 registers)
#endif
template <bool STRICT>
__global__ void __launch_bounds__(kTileThreads, OSB_K3_CTAS) k_blend(const uint32_t* __restrict__ inst_gid,
                                                           uint2* __restrict__ ranges, PreprocessOut pp, int W,
                                                           int H, int tiles_x, float bg0, float bg1, float bg2,
                                                           FrameBuffers fb, int tile0) {
    pdl_begin();
    // CTA-cooperative walk: the 8 warps stage 512 entries at once (two per thread, each entry once
    // per tile instead of once per warp, with a 16-bit reach mask for all quarters), then every warp
    // blends the 16 sub-chunks in list order; one barrier pair per 512 entries (256: 0.56 ms,
    // 512: 0.51 ms, 768: 0.53 ms — the barrier wait of the slowest warp is paid less often).
    constexpr int kPer = OSB_K3_PER;                      // entries staged per thread per round
    constexpr int kChunk = kPer * kTileThreads;   // entries per round (one barrier pair)
    constexpr int kSubs = kChunk / 32;
    __shared__ WarpStage stage[kSubs];
    __shared__ uint16_t s_mask[kChunk];
    const int tile = tile0 + block_tile(tiles_x, (H + kTile - 1) / kTile);  // tile0: banded launches
    const int tx = tile % tiles_x, ty = tile / tiles_x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const WarpPixel wp = warp_pixel(warp, lane);
    const int lx = wp.lx, ly = wp.ly;
    const int px = tx * kTile + lx, py = ty * kTile + ly;
    const bool inside = px < W && py < H;
    uint2 range = ranges[tile];
    if (range.x > range.y) {  // an empty tile of the fused tile sort ({~0u, 0}): stored back as {0, 0}
        range = make_uint2(0u, 0u);
        if (threadIdx.x == 0) ranges[tile] = range;
    }
    const double width = W;
    const double xc = tx * kTile + 8.0, yc = ty * kTile + 8.0;
    float lxo = lx - 7.5f, lyo = ly - 7.5f;
    // opaque to the compiler: kept in registers instead of being rematerialized from tid in the loop
    asm volatile("mov.b32 %0, %0;" : "+f"(lxo));
    asm volatile("mov.b32 %0, %0;" : "+f"(lyo));
    const float halfW = 0.5f * W, fW = static_cast<float>(W);
    const uint32_t stage_s = pinned_smem_base(stage);
    const float2 nlo = make_float2(-lxo, -lyo);

    float T = 1.0f, c2 = 0.0f;
    float2 c01 = make_float2(0.0f, 0.0f);  // (c0, c1), updated with one packed FFMA2
    double T64 = 1.0;
    float Terr = 0.0f;  // bound on alpha-error propagation into T (exact mode: not needed)
    bool exact = false;
    int contrib = 0, last = 0;
    int stop_at = static_cast<int>(range.y - range.x);  // entries evaluated (work counting)
    bool done = !inside;

    const int t = threadIdx.x;
#ifdef OSB_K3_STATS
    unsigned long long st[5] = {0, 0, 0, 0, 0};
#endif
    uint32_t gid_next[kPer];  // ids one round ahead
#pragma unroll
    for (int e = 0; e < kPer; ++e)
        gid_next[e] = range.x + t + e * kTileThreads < range.y ? inst_gid[range.x + t + e * kTileThreads] : 0u;
    for (uint32_t cbase = range.x; cbase < range.y; cbase += kChunk) {
        // every pixel of the tile has terminated (no barrier before the first round: nothing staged yet)
        if (cbase != range.x && !__syncthreads_or(!done)) break;
#pragma unroll
        for (int e = 0; e < kPer; ++e) {
            const uint32_t idx = cbase + t + e * kTileThreads;
            const uint32_t gid = gid_next[e];
            gid_next[e] = idx + kChunk < range.y ? inst_gid[idx + kChunk] : 0u;
            uint32_t m = 0u;
            if (idx < range.y) {
                const float4* s4 = reinterpret_cast<const float4*>(pp.splat + gid);
                m = stage_record16<OSB_K3_ELLIPSE>(stage[warp + e * kTileWarps], lane, gid, pp.pxy[gid], s4[0], s4[1], s4[2], xc,
                                   yc, width);
            }
            s_mask[t + e * kTileThreads] = static_cast<uint16_t>(m);
        }
        __syncthreads();
      for (int sub = 0; sub < kSubs; ++sub) {
        const uint32_t base = cbase + 32 * sub;
        if (base >= range.y || __all_sync(0xffffffffu, done)) break;
        const StageRef ws{stage_s + static_cast<uint32_t>(sub * sizeof(WarpStage))};
        const int kofs = static_cast<int>(base - range.x) + 1;  // 1-based list position of entry j: kofs + j
        const uint32_t mk = s_mask[32 * sub + lane];
        const uint32_t bal0 = __ballot_sync(0xffffffffu, (mk >> (2 * warp)) & 1u);
        const uint32_t bal1 = __ballot_sync(0xffffffffu, (mk >> (2 * warp + 1)) & 1u);
        uint32_t bal = wp.half ? bal1 : bal0;  // this half-warp's entries; lanes loop independently
        // A lane whose FP32 transmittance lands inside the T band parks the entry (pend) and leaves
        // the loop; the warp then replays each parked pixel's prefix cooperatively (warp_replay_T:
        // 32 entries evaluated in parallel, product in list order) and the lane resumes.
        const bool seam = __any_sync(0xffffffffu, ws.b(lane).w < 0.0f);  // a seam-straddling entry here
        bool pend = false, p_unc = false;
        int pj = 0;
        double p_a64 = 0.0;
        for (;;) {
            // the lane loop, specialised for sub-chunks without seam-straddling entries (measured:
            // 0.583 -> 0.560 ms; a second specialisation for warps without a pixel in exact mode
            // spilled and lost that gain again)
            auto lanes = [&](auto seam_tag) {
                constexpr bool SEAM = decltype(seam_tag)::value;
                while (bal != 0u && !done && !pend) {
                    const int j = __ffs(bal) - 1;
                    bal &= bal - 1u;
#ifdef OSB_K3_STATS
                    {
                        const uint32_t am = __activemask();
                        if (lane == __ffs(am) - 1) {
                            st[0] += 1;  // warp iterations
                            st[4] += ((am & 0xFFFFu) != 0u) + ((am >> 16) != 0u);  // live halves
                        }
                        st[1] += 1;  // lanes evaluating
                    }
#endif
                    const float4 A = ws.a(j);
                    const float4 B = ws.b(j);
                    float2 d;
                    float power;
                    bool unc;
                    if (!pair_power2<SEAM>(A, B, nlo, halfW, fW, d, power, unc)) continue;
#ifdef OSB_K3_STATS
                    st[2] += 1;  // lanes past the power test
#endif
                    const float4 Cc = ws.c(j);
                    float alpha;
                    double a64 = 0.0;
                    if (unc || exact) {
                        Pair64 p;
                        if (!pair_slow(ws.gid(j), px, py, width, pp.pxy, pp.conic_o, &p)) continue;
                        a64 = p.alpha;
                        alpha = static_cast<float>(a64);
                    } else {
                        alpha = fminf(0.99f, Cc.w * ex2_approx(-power * kLog2e));
                    }
                    float w;
                    if (!exact) {
                        const float one_m = 1.0f - alpha;
                        const float Tn = T * one_m;
                        bool near;
                        float lo;
                        if (STRICT) {
                            // relative error bound of the FP32 T (common.cuh): alpha / (1 - alpha) x
                            // alpha's relative error bound; the per-step rounding term from `contrib`
                            float inv;
                            asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(inv) : "f"(one_m));
                            const float dlt = fabsf(B.w);
                            Terr = __fmaf_rn(alpha * inv, __fmaf_rn(dlt, 1.001f + dlt, kAlphaErr), Terr);
                            // Terr <= 0.2 and < 4e5 steps keep e <= 0.25: T_next >= kTPre is then certain
                            near = Tn < kTPre || Terr > 0.2f;
                            lo = 0.0f;
                            if (near) {
                                const float e = __fmaf_rn(static_cast<float>(contrib + 1), kTStep, Terr);
                                const float em = __fmaf_rn(2.0f * e, e, e) + kTMargin;
                                near = Tn < 1e-4f * (1.0f + em);
                                lo = 1e-4f * (1.0f - em);
                            }
                        } else {
                            near = Tn < kTHi;
                            lo = kTLo;
                        }
                        if (near) {
                            if (Tn < lo) {
                                done = true;
                                stop_at = kofs + j;
                                break;
                            }
                            pend = true;  // inside the band: decide in FP64 after an exact replay
                            pj = j;
                            p_unc = unc;
                            p_a64 = a64;
                            break;
                        }
                        w = alpha * T;
                        T = Tn;
                    } else {
                        const double Tn64 = T64 * (1.0 - a64);
                        if (Tn64 < kTStop) {
                            done = true;
                            stop_at = kofs + j;
                            break;
                        }
                        w = static_cast<float>(a64 * T64);
                        T64 = Tn64;
                        T = static_cast<float>(Tn64);
                    }
                    c01 = __ffma2_rn(make_float2(Cc.x, Cc.y), make_float2(w, w), c01);
                    c2 = __fmaf_rn(Cc.z, w, c2);
#ifdef OSB_K3_STATS
                    st[3] += 1;  // lanes contributing
#endif
                    ++contrib;
                    last = kofs + j;
                }
            };
            if (seam) lanes(std::true_type{});
            else lanes(std::false_type{});
            uint32_t pm = __ballot_sync(0xffffffffu, pend);
            if (pm == 0u) break;
            while (pm != 0u) {
                const int L = __ffs(pm) - 1;
                pm &= pm - 1u;
                const uint32_t kL = __shfl_sync(0xffffffffu, base + pj, L);
                const int pxL = __shfl_sync(0xffffffffu, px, L), pyL = __shfl_sync(0xffffffffu, py, L);
                const double t = warp_replay_T(inst_gid, range.x, kL, pxL, pyL, width, pp.pxy, pp.conic_o, lane);
                if (lane == L) T64 = t;
            }
            if (pend) {
                pend = false;
                double a64 = p_a64;
                if (!p_unc) {
                    Pair64 p;
                    pair_slow(ws.gid(pj), px, py, width, pp.pxy, pp.conic_o, &p);
                    a64 = p.alpha;
                }
                const double Tn64 = T64 * (1.0 - a64);
                if (Tn64 < kTStop) {
                    done = true;
                    stop_at = kofs + pj;
                } else {
                    exact = true;
                    const float4 Cc = ws.c(pj);
                    const float w = static_cast<float>(a64 * T64);
                    T64 = Tn64;
                    T = static_cast<float>(Tn64);
                    c01 = __ffma2_rn(make_float2(Cc.x, Cc.y), make_float2(w, w), c01);
                    c2 = __fmaf_rn(Cc.z, w, c2);
                    ++contrib;
                    last = kofs + pj;
                }
            }
        }
        __syncwarp();
      }
        // no barrier here: the next round's __syncthreads_or is the one that orders this round's
        // stage reads before the restaging
    }
#ifdef OSB_K3_STATS
    for (int q = 0; q < 5; ++q) atomicAdd(&g_k3_stats[q], st[q]);
#endif
    if (inside) {
        const size_t pix = static_cast<size_t>(py) * W + px;
        const size_t plane = static_cast<size_t>(W) * H;
        fb.rgb[pix] = __fmaf_rn(T, bg0, c01.x);
        fb.rgb[plane + pix] = __fmaf_rn(T, bg1, c01.y);
        fb.rgb[2 * plane + pix] = __fmaf_rn(T, bg2, c2);
        fb.T[pix] = T;
        fb.contrib[pix] = contrib;
        fb.last[pix] = last;
        if (fb.visited) fb.visited[pix] = stop_at;
    }
}

__global__ void k_work_count(const int* __restrict__ visited, const int* __restrict__ last, int pixels,
                             unsigned long long* __restrict__ out) {
    unsigned long long a = 0, b = 0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < pixels; i += gridDim.x * blockDim.x) {
        a += static_cast<unsigned long long>(visited[i]);
        b += static_cast<unsigned long long>(last[i]);
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        a += __shfl_down_sync(0xffffffffu, a, off);
        b += __shfl_down_sync(0xffffffffu, b, off);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(out, a);
        atomicAdd(out + 1, b);
    }
}

}  // namespace

namespace {
__global__ void __launch_bounds__(256) k_planar_to_hwc_f64(const float* __restrict__ rgb, size_t plane, size_t p0,
                                                           size_t p1, double* __restrict__ out) {
    for (size_t i = p0 + blockIdx.x * 256ull + threadIdx.x; i < p1; i += static_cast<size_t>(gridDim.x) * 256ull) {
        out[3 * i] = rgb[i];
        out[3 * i + 1] = rgb[plane + i];
        out[3 * i + 2] = rgb[2 * plane + i];
    }
}
}  // namespace

void launch_planar_to_hwc_f64(const float* rgb, size_t plane, double* out, cudaStream_t s, size_t p0, size_t p1) {
    if (p1 == static_cast<size_t>(-1)) p1 = plane;
    if (p1 <= p0) return;
    size_t blocks = (p1 - p0 + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    k_planar_to_hwc_f64<<<static_cast<int>(blocks), 256, 0, s>>>(rgb, plane, p0, p1, out);
    OSB_LAUNCHED(1);
}

void launch_work_count(const FrameBuffers& fb, int pixels, unsigned long long* out, cudaStream_t s) {
    OSB_CUDA_CHECK(cudaMemsetAsync(out, 0, 16, s));
    if (pixels <= 0 || !fb.visited) return;
    k_work_count<<<296, 256, 0, s>>>(fb.visited, fb.last, pixels, out);
    OSB_LAUNCHED(1);
}

void launch_blend(const uint32_t* inst_gid, uint2* ranges, const PreprocessOut& pp, int W, int H, int tiles_x,
                  int tiles_y, const float bg[3], const FrameBuffers& fb, cudaStream_t s, bool strict, int row0,
                  int row1) {
    if (row1 < 0 || row1 > tiles_y) row1 = tiles_y;
    const int tile0 = row0 * tiles_x, tiles = (row1 - row0) * tiles_x;
    if (tiles <= 0) return;
    if (strict)
        k_blend<true><<<tiles, kTileThreads, 0, s>>>(inst_gid, ranges, pp, W, H, tiles_x, bg[0], bg[1], bg[2], fb,
                                                     tile0);
    else
        k_blend<false><<<tiles, kTileThreads, 0, s>>>(inst_gid, ranges, pp, W, H, tiles_x, bg[0], bg[1], bg[2], fb,
                                                      tile0);
    OSB_LAUNCHED(1);
}

#ifdef OSB_K3_STATS
extern "C" __attribute__((visibility("default"))) void osb_k3_stats(unsigned long long* out, int reset) {
    cudaMemcpyFromSymbol(out, g_k3_stats, sizeof(unsigned long long) * 5);
    if (reset) {
        unsigned long long z[5] = {0, 0, 0, 0, 0};
        cudaMemcpyToSymbol(g_k3_stats, z, sizeof(z));
    }
}
#endif

}  // namespace osb
