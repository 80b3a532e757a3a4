// backward.cu — K4a (per-pixel, reverse order) and K4b (per-Gaussian chain rule, FP64).
//
// K4a replaces backward() pass 1 + pass 2 (proj/src/gradients.cpp:96-169): same CTA/tile layout
// and half-warp culling as K3 (pair.cuh), each 4x4 quarter walking its entries back to front from
// each pixel's last_contrib. The 9 per-entry accumulators (d_colour 3, d_opacity, d_p 2, d_conic 3)
// of a quarter's pixels are combined with a reduce-scatter shuffle tree inside the half-warp and
// added by one red.global.add.f32 per value; when the warp has at most 14 contributing lanes
// (warp-uniform choice) they add directly (2 x red.v4 + 1 each). Pair decisions are the forward's;
// the 0.99 clamp gate (gradients.cpp:146) has its own FP64 guard.
//
// K4b replaces pass 3 (gradients.cpp:173-295): one thread per visible Gaussian, FP64 internals,
// re-derives t, J, Sigma and the conic with the same device code as K1 and accumulates the raw
// parameter gradients into the flat FP32 plane buffer (allreduce-able as one tensor).
#include <type_traits>

#include "kernels.h"
#include "pair.cuh"
#include "project.cuh"

namespace osb {

namespace {

#ifdef OSB_K4A_STATS
// Instrumented build only (scripts/k4a_stats.py): K4a loop statistics per launch.
__device__ unsigned long long g_k4a_stats[8];
#define OSB_STAT(i, v) (st[i] += (v))
#else
#define OSB_STAT(i, v) ((void)0)
#endif

__device__ __forceinline__ void red_add_v4(float4* addr, float a, float b, float c, float d) {
    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(addr), "f"(a), "f"(b), "f"(c), "f"(d)
                 : "memory");
}
__device__ __forceinline__ void red_add(float* addr, float a) {
    asm volatile("red.global.add.f32 [%0], %1;" ::"l"(addr), "f"(a) : "memory");
}

// Reduce-scatter of 9 values inside each 16-lane half (xor 8, 4, 2, 1; 9 -> 5 -> 3 -> 2 -> 1 values
// per lane, 10 shuffles): both halves reduce their own entry at once; afterwards lane l of a half
// holds the half's sum of value *idx (-1: padding).
__device__ __forceinline__ float half_reduce9(const float (&v)[9], int lane, int* idx) {
    const bool b3 = lane & 8, b2 = lane & 4, b1 = lane & 2, b0 = lane & 1;
    // the adds of a stage issue in pairs as packed FADD2 (each half rounded like the scalar add)
    float k[5], r[5];
#pragma unroll
    for (int i = 0; i < 5; ++i) {
        const float lo = v[i];
        const float hi = i + 5 < 9 ? v[i + 5] : 0.0f;
        k[i] = b3 ? hi : lo;
        r[i] = __shfl_xor_sync(0xffffffffu, b3 ? lo : hi, 8);
    }
    float a[5];
    {
        const float2 s01 = __fadd2_rn(make_float2(k[0], k[1]), make_float2(r[0], r[1]));
        const float2 s23 = __fadd2_rn(make_float2(k[2], k[3]), make_float2(r[2], r[3]));
        a[0] = s01.x; a[1] = s01.y; a[2] = s23.x; a[3] = s23.y;
        a[4] = k[4] + r[4];
    }
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        const float lo = a[i];
        const float hi = i + 3 < 5 ? a[i + 3] : 0.0f;
        k[i] = b2 ? hi : lo;
        r[i] = __shfl_xor_sync(0xffffffffu, b2 ? lo : hi, 4);
    }
    float c[3];
    {
        const float2 s01 = __fadd2_rn(make_float2(k[0], k[1]), make_float2(r[0], r[1]));
        c[0] = s01.x; c[1] = s01.y;
        c[2] = k[2] + r[2];
    }
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        const float lo = c[i];
        const float hi = i + 2 < 3 ? c[i + 2] : 0.0f;
        k[i] = b1 ? hi : lo;
        r[i] = __shfl_xor_sync(0xffffffffu, b1 ? lo : hi, 2);
    }
    float e[2];
    {
        const float2 s01 = __fadd2_rn(make_float2(k[0], k[1]), make_float2(r[0], r[1]));
        e[0] = s01.x; e[1] = s01.y;
    }
    const float f = (b0 ? e[1] : e[0]) + __shfl_xor_sync(0xffffffffu, b0 ? e[0] : e[1], 1);
    const int ic = (b1 ? 2 : 0) + (b0 ? 1 : 0);
    const int ia = (b2 ? 3 : 0) + ic;
    const bool pad = (b1 && b0) || (b2 && ic == 2) || (b3 && ia == 4);
    *idx = pad ? -1 : (b3 ? 5 : 0) + ia;
    return f;
}

// FP64 evaluation of instance `gid` at this thread's pixel (rasterizer.cpp:128-134) for K4a:
// returns {alpha, g} with alpha = -1 when the pair does not contribute in FP64 and g negated when the
// 0.99 clamp gate (gradients.cpp:146, o g < 0.99) is closed. Out of line: called for < 0.1 % of pairs.
static __device__ __noinline__ float2 k4a_slow(uint32_t gid) {
    int px, py;
    slow_pixel(px, py);
    const double2 pc = s_slow.pxy[gid];
    const double4 co = s_slow.conic_o[gid];
    double g, alpha;
    if (!pair_fp64(pc.x, pc.y, co.x, co.y, co.z, co.w, px + 0.5, py + 0.5, s_slow.width, &g, &alpha))
        return make_float2(-1.0f, 0.0f);
    const float gf = static_cast<float>(g);
    return make_float2(static_cast<float>(alpha), co.w * g < kAlphaMax ? gf : -gf);
}

// BG: a non-black background adds the -T_final / (1 - alpha) * (bg . dL/dC) term (gradients.cpp:141).
//
// Hot loop (one entry per half-warp per iteration, back to front): branch-free for the common case.
// Every lane evaluates the staged entry its half selected; a lane that does not contribute (no entry
// left, entry at or past its last_contrib, certain FP32 skip, FP64 skip) carries alpha = 0 and g = 0,
// which leaves T_acc and the suffix colour bit-identical (x * rcp(1) = x, fma(c, -0, s * 1) = s)
// and makes all nine accumulated values zero. Only the FP64 fallback (pairs inside the guard band,
// or the 0.99 clamp gate of a near-opaque splat) branches, warp-uniformly.
template <bool BG>
#ifndef OSB_K4A_PER
#define OSB_K4A_PER 2  // entries staged per thread per round (512-entry rounds)
#endif
#ifndef OSB_K4A_TOTAL
#define OSB_K4A_TOTAL 14  // tree when the warp has more contributing lanes (0: either half > OSB_K4A_DIRECT)
#endif
#ifndef OSB_K4A_DIRECT
#define OSB_K4A_DIRECT 10  // a quarter's entry with at most this many contributing pixels: direct atomics
#endif
#ifndef OSB_K4A_CTAS
#define OSB_K4A_CTAS 4  // CTAs per SM (64 registers)
#endif
__global__ void __launch_bounds__(kTileThreads, OSB_K4A_CTAS) k_backward_pixels(const uint32_t* __restrict__ inst_gid,
                                                                     const uint2* __restrict__ ranges, PreprocessOut pp,
                                                                     int W, int H, int tiles_x, float bg0, float bg1,
                                                                     float bg2, FrameBuffers fb,
                                                                     const float* __restrict__ d_image,
                                                                     float4* __restrict__ acc) {
    pdl_begin();
    // CTA-cooperative walk (as K3): 512 entries staged at once with 16-quarter reach masks, every
    // warp then walks the 16 sub-chunks back to front.
    constexpr int kPer = OSB_K4A_PER;                      // entries staged per thread per round
    constexpr int kChunk = kPer * kTileThreads;   // entries per round (one barrier pair)
    constexpr int kSubs = kChunk / 32;
    __shared__ WarpStage stage[kSubs];
    __shared__ uint16_t s_mask[kChunk];
    __shared__ int s_last[kTileWarps];
    const int tile = block_tile(tiles_x, (H + kTile - 1) / kTile);
    const int tx = tile % tiles_x, ty = tile / tiles_x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const WarpPixel wp = warp_pixel(warp, lane);
    const int lx = wp.lx, ly = wp.ly;
    const int px = tx * kTile + lx, py = ty * kTile + ly;
    const bool inside = px < W && py < H;
    const uint2 range = ranges[tile];
    const double width = W;
    const double xc = tx * kTile + 8.0, yc = ty * kTile + 8.0;
    float lxo = lx - 7.5f, lyo = ly - 7.5f;
    asm volatile("mov.b32 %0, %0;" : "+f"(lxo));
    asm volatile("mov.b32 %0, %0;" : "+f"(lyo));
    const float halfW = 0.5f * W, fW = static_cast<float>(W);
    const float2 nlo = make_float2(-lxo, -lyo);
    const size_t pix = static_cast<size_t>(py) * W + px;
    const size_t plane = static_cast<size_t>(W) * H;
    const int last = inside ? fb.last[pix] : 0;
    const float T_final = inside ? fb.T[pix] : 0.0f;
    const float dl0 = inside ? d_image[pix] : 0.0f;
    const float dl1 = inside ? d_image[plane + pix] : 0.0f;
    const float2 dl01 = make_float2(dl0, dl1);
    const float dl2 = inside ? d_image[2 * plane + pix] : 0.0f;
    const float bg_dot = bg0 * dl0 + bg1 * dl1 + bg2 * dl2;
    // this warp only walks the list up to its own furthest last_contrib
    const int max_last = static_cast<int>(__reduce_max_sync(0xffffffffu, static_cast<unsigned>(last)));
    const uint32_t stage_s = pinned_smem_base(stage);

    float T_acc = T_final;
    // negated suffix colour (-s): (Cc - s) is then one packed add; ns01 = (-s0, -s1)
    float2 ns01 = make_float2(0.0f, 0.0f);
    float ns2 = 0.0f;

    // Each 16-lane half owns a 4x4 pixel quarter and walks the entries that can reach it (the same
    // half-warp culling as K3), back to front; the halves reduce their (different) entries at once.
    const uint32_t halfmask = wp.half ? 0xFFFF0000u : 0x0000FFFFu;
    if (lane == 0) s_last[warp] = max_last;
    if (threadIdx.x == 0) s_slow = SlowCtx{pp.pxy, pp.conic_o, width, tiles_x, tile};
    __syncthreads();
    int cta_last = 0;
#pragma unroll
    for (int w = 0; w < kTileWarps; ++w) cta_last = max(cta_last, s_last[w]);
    const int t = threadIdx.x;
#ifdef OSB_K4A_STATS
    unsigned long long st[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#endif
    for (int hi = cta_last; hi > 0; hi -= kChunk) {
        const int lo = hi > kChunk ? hi - kChunk : 0;
        OSB_STAT(7, lane == 0 ? static_cast<unsigned long long>(hi - lo) : 0ull);
#pragma unroll
        for (int e = 0; e < kPer; ++e) {
            const int i = lo + t + e * kTileThreads;
            uint32_t m = 0u;
            if (i < hi) {
                const uint32_t gid = inst_gid[range.x + i];
                const float4* s4 = reinterpret_cast<const float4*>(pp.splat + gid);
                m = stage_record16<true>(stage[warp + e * kTileWarps], lane, gid, pp.pxy[gid], s4[0], s4[1], s4[2], xc, yc,
                                   width);
            } else {
                // finite filler: lanes with no entry left evaluate slot 31 with alpha forced to 0
                WarpStage& w = stage[warp + e * kTileWarps];
                w.a[lane] = w.b[lane] = w.c[lane] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
                w.gid[lane] = 0u;
            }
            s_mask[t + e * kTileThreads] = static_cast<uint16_t>(m);
        }
        __syncthreads();
      for (int sub = kSubs - 1; sub >= 0; --sub) {
        const int sbase = lo + 32 * sub;
        if (sbase >= hi || sbase >= max_last) continue;  // no pixel of this warp reaches these entries
        const StageRef ws{stage_s + static_cast<uint32_t>(sub * sizeof(WarpStage))};
        const uint32_t mk = s_mask[32 * sub + lane];
        const uint32_t bal0 = __ballot_sync(0xffffffffu, (mk >> (2 * warp)) & 1u);
        const uint32_t bal1 = __ballot_sync(0xffffffffu, (mk >> (2 * warp + 1)) & 1u);
        uint32_t bal = wp.half ? bal1 : bal0;
        // entry j of this sub-chunk lies before this pixel's last_contrib iff j < kl
        const uint32_t kl = static_cast<uint32_t>(min(max(last - sbase, 0), 32));
        OSB_STAT(0, 1);
        // the per-pixel seam wrap only in sub-chunks that hold a seam-straddling entry (B.w < 0)
        auto walk = [&](auto seam_tag) {
            constexpr bool SEAM = decltype(seam_tag)::value;
            while (__any_sync(0xffffffffu, bal != 0u)) {  // back to front; warp-uniform (the reduction needs all lanes)
                const uint32_t j = bfind_u32(bal);  // ~0u once this half has no entry left
                bal &= below_u32(j);  // j is bal's highest set bit: clear it (~0u: bal is already 0)
                const uint32_t jj = j & 31u;
                OSB_STAT(1, 1);
                const float4 A = ws.a(jj);
                const float4 B = ws.b(jj);
                const float4 Cc = ws.c(jj);
                // FP32 power, exactly pair_power2's instructions (K3 makes the same decisions)
                float2 d = __fadd2_rn(make_float2(A.x, A.y), nlo);
                bool unc = false;
                if (SEAM && B.w < 0.0f) {
                    if (d.x > halfW) d.x -= fW;
                    else if (d.x < -halfW) d.x += fW;
                    unc = fabsf(fabsf(d.x) - halfW) < 0.01f;
                }
                const float2 q = __fmul2_rn(make_float2(A.z, A.w), d);
                const float bdx = B.x * d.x;
                const float power = __fmaf_rn(q.x, d.x, __fmaf_rn(q.y, d.y, bdx * d.y));
                // candidate: an entry of this half before the pixel's last_contrib that is not a certain skip
                const bool cand = j < kl && (power <= B.z || unc);
                unc = unc || power < fabsf(B.w) || power > B.y;
                float g = ex2_approx(-power * kLog2e);
                const float og = Cc.w * g;
                float alpha = fminf(0.99f, og);
                // 0.99 clamp gate: certain in FP32 unless a near-opaque splat (o >= 0.98) lands inside its
                // guard band — checked only behind the rare-path vote
                bool gate = og < 0.99f;
                bool has = cand;
                if (__any_sync(0xffffffffu, cand && (unc || Cc.w >= 0.98f))) {
                    const bool gchk = Cc.w >= 0.98f && fabsf(og - 0.99f) <= 0.99f * (1.5f * fabsf(B.w) + 1e-6f);
                    if (cand && (unc || gchk)) {
                        const float2 r = k4a_slow(ws.gid(jj));
                        if (unc) {
                            has = r.x >= 0.0f;
                            alpha = r.x;
                            g = fabsf(r.y);
                        }
                        gate = r.y > 0.0f;
                    }
                }
                OSB_STAT(5, __popc(__ballot_sync(0xffffffffu, j < kl)));
                alpha = has ? alpha : 0.0f;
                g = has && gate ? g : 0.0f;
                const float one_m = 1.0f - alpha;
                // 1 - alpha is in [0.01, 1]: MUFU.RCP directly (what __fdividef(1, x) computes there,
                // without its range-scaling instructions); rcp(1) = 1 exactly
                float inv;
                asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(inv) : "f"(one_m));
                T_acc = T_acc * inv;
                const float wb = alpha * T_acc;
                const float2 v01 = __fmul2_rn(dl01, make_float2(wb, wb));
                const float v2 = dl2 * wb;
                const float2 cs = __fadd2_rn(make_float2(Cc.x, Cc.y), ns01);  // Cc - s
                float d_alpha = cs.x * dl01.x;
                d_alpha = __fmaf_rn(cs.y, dl01.y, d_alpha);
                d_alpha = __fmaf_rn(Cc.z + ns2, dl2, d_alpha);
                d_alpha = d_alpha * T_acc;
                if (BG) d_alpha = d_alpha - (T_final * inv) * bg_dot;
                // suffix (colour of everything behind) now includes this entry:
                // (-s) = fma(Cc, -alpha, (-s) (1 - alpha)), the exact negation of fma(Cc, alpha, s (1 - alpha))
                const float nalpha = -alpha;
                ns01 = __ffma2_rn(make_float2(Cc.x, Cc.y), make_float2(nalpha, nalpha),
                                  __fmul2_rn(ns01, make_float2(one_m, one_m)));
                ns2 = __fmaf_rn(Cc.z, nalpha, ns2 * one_m);
                // dL/dpower times d, d d^T: K4b applies the conic once per Gaussian
                // (d_p = Q sum(dL/dpower d)) and the 1/2 of the conic diagonal
                const float v3 = g * d_alpha;
                const float d_power = -Cc.w * v3;
                const float2 v45 = __fmul2_rn(d, make_float2(d_power, d_power));
                const float2 v67 = __fmul2_rn(d, make_float2(v45.x, v45.x));
                const float v8 = v45.y * d.y;
                const uint32_t hb_all = __ballot_sync(0xffffffffu, has);
                OSB_STAT(6, __popc(hb_all));
                // (no early `continue` when no lane contributes: 99.4 % of the iterations have a
                // contributor, and with hb_all = 0 nothing below adds anything)
                OSB_STAT(2, hb_all != 0u ? 1 : 0);
                const uint32_t hb = hb_all & halfmask;  // this half's contributing lanes
                float* a = reinterpret_cast<float*>(acc + 3 * static_cast<size_t>(ws.gid(jj)));
                // up to 10 contributing pixels of this quarter add directly (3 red instructions per
                // warp, the L2 absorbs the per-lane atomics); more are cheaper through the shuffle tree
                // (measured: always-tree 1.32 ms, <=10 direct 1.21 ms, always-direct 1.70 ms; with the
                // branch-free loop: <=6 direct 0.988, <=10 0.954; one or two butterfly levels then direct
                // adds by the group leaders 1.177 / 1.027; the tree's sums gathered into two red.v4 + one
                // scalar per half 1.055 — the L2 absorbs nine scalar reds better than the extra shuffles)
                // warp-uniform choice: when the warp has more than OSB_K4A_TOTAL contributing lanes
                // both halves go through the tree (its shuffles serve both halves at once, so the
                // other half's reduction is free and saves its direct atomics)
#if OSB_K4A_TOTAL
                // measured: the warp's total > 8 / 10 / 12 / 14 / 16 / 20: 0.848 / 0.832 / 0.820 /
                // 0.814 / 0.829 / 0.954 ms; either half > 10: 0.835 ms
                const bool multi = __popc(hb_all) > OSB_K4A_TOTAL;
#else
                const bool multi = __any_sync(0xffffffffu, __popc(hb) > OSB_K4A_DIRECT);
#endif
                if (!multi) {
                    if (has) {
                        red_add_v4(reinterpret_cast<float4*>(a), v01.x, v01.y, v2, v3);
                        red_add_v4(reinterpret_cast<float4*>(a) + 1, v45.x, v45.y, v67.x, v67.y);
                        red_add(a + 8, v8);
                    }
                } else {
                    OSB_STAT(3, 1);
                    const float v[9] = {v01.x, v01.y, v2, v3, v45.x, v45.y, v67.x, v67.y, v8};
                    int idx;
                    const float sum = half_reduce9(v, lane, &idx);
                    if (hb != 0u && idx >= 0) red_add(a + idx, sum);
                }
            }
        };
        if (__any_sync(0xffffffffu, ws.b(lane).w < 0.0f)) walk(std::true_type{});
        else walk(std::false_type{});
        __syncwarp();
      }
        __syncthreads();  // the stage is rewritten by the next chunk
    }
#ifdef OSB_K4A_STATS
    if (lane == 0)
        for (int i = 0; i < 8; ++i) atomicAdd(&g_k4a_stats[i], st[i]);
#endif
}

// Gradient plane update: OVERWRITE (the buffer is logically zero: first view after Adam or a
// non-accumulating backward) stores, otherwise adds (multi-view accumulation) with a
// fire-and-forget red.global.add: one thread owns each element within a launch, so the sum is the
// same single FP32 add as a read-modify-write, without 59 load -> store round trips in series (the
// compiler cannot prove the planes distinct and would serialise them).
template <bool OVERWRITE, typename R>
__device__ __forceinline__ void put_grad(float* __restrict__ G, int stride, int plane, int gid, R v) {
    float* p = G + static_cast<size_t>(plane) * stride + gid;
    if (OVERWRITE) *p = static_cast<float>(v);
    else red_add(p, static_cast<float>(v));
}

// One SH basis function of the backward (gradients.cpp:202-207): d_sh_i = dl_color * b_i and
// d_dir += db_i * (c_i . dl_color), with b_i / db_i from scene.cpp:45-92. Evaluated in FP32
// (R = float): the basis and its gradient are well conditioned (|dir| = 1), the pre-clamp colour
// gate comes exactly from K1, and the results stay far inside the 1e-3 gradient tolerance; the
// cancellation-prone geometry chain below stays FP64.
template <typename R, bool OVERWRITE>
struct ShBack {
    const float* P;
    float* G;
    int stride, gid;
    Planes pl;
    R dlc[3];
    R dd[3];
    __device__ __forceinline__ void basis(int i, R b, R gx, R gy, R gz) {
        const R c0 = static_cast<R>(__ldg(P + static_cast<size_t>(pl.sh(i, 0)) * stride + gid));
        const R c1 = static_cast<R>(__ldg(P + static_cast<size_t>(pl.sh(i, 1)) * stride + gid));
        const R c2 = static_cast<R>(__ldg(P + static_cast<size_t>(pl.sh(i, 2)) * stride + gid));
        put_grad<OVERWRITE>(G, stride, pl.sh(i, 0), gid, dlc[0] * b);
        put_grad<OVERWRITE>(G, stride, pl.sh(i, 1), gid, dlc[1] * b);
        put_grad<OVERWRITE>(G, stride, pl.sh(i, 2), gid, dlc[2] * b);
        const R cdot = c0 * dlc[0] + c1 * dlc[1] + c2 * dlc[2];
        dd[0] += gx * cdot;
        dd[1] += gy * cdot;
        dd[2] += gz * cdot;
    }
};

template <int DEG, typename R, bool OVERWRITE>
__device__ __forceinline__ void sh_backward(ShBack<R, OVERWRITE>& s, const R* d) {
    constexpr R C0 = static_cast<R>(0.28209479177387814);
    constexpr R C1 = static_cast<R>(0.4886025119029199);
    constexpr R C20 = static_cast<R>(1.0925484305920792), C21 = static_cast<R>(-1.0925484305920792),
                C22 = static_cast<R>(0.31539156525252005), C23 = static_cast<R>(-1.0925484305920792),
                C24 = static_cast<R>(0.5462742152960396);
    constexpr R C30 = static_cast<R>(-0.5900435899266435), C31 = static_cast<R>(2.890611442640554),
                C32 = static_cast<R>(-0.4570457994644658), C33 = static_cast<R>(0.3731763325901154),
                C34 = static_cast<R>(-0.4570457994644658), C35 = static_cast<R>(1.445305721320277),
                C36 = static_cast<R>(-0.5900435899266435);
    constexpr R k0 = 0, k2 = 2, k3 = 3, k4 = 4, k6 = 6, k8 = 8;
    const R x = d[0], y = d[1], z = d[2];
    s.basis(0, C0, k0, k0, k0);
    if (DEG < 1) return;
    s.basis(1, -C1 * y, k0, -C1, k0);
    s.basis(2, C1 * z, k0, k0, C1);
    s.basis(3, -C1 * x, -C1, k0, k0);
    if (DEG < 2) return;
    const R xx = x * x, yy = y * y, zz = z * z;
    s.basis(4, C20 * x * y, C20 * y, C20 * x, k0);
    s.basis(5, C21 * y * z, k0, C21 * z, C21 * y);
    s.basis(6, C22 * (k2 * zz - xx - yy), -k2 * C22 * x, -k2 * C22 * y, k4 * C22 * z);
    s.basis(7, C23 * x * z, C23 * z, k0, C23 * x);
    s.basis(8, C24 * (xx - yy), k2 * C24 * x, -k2 * C24 * y, k0);
    if (DEG < 3) return;
    s.basis(9, C30 * y * (k3 * xx - yy), C30 * k6 * x * y, C30 * (k3 * xx - k3 * yy), k0);
    s.basis(10, C31 * x * y * z, C31 * y * z, C31 * x * z, C31 * x * y);
    s.basis(11, C32 * y * (k4 * zz - xx - yy), -k2 * C32 * x * y, C32 * (k4 * zz - xx - k3 * yy), k8 * C32 * y * z);
    s.basis(12, C33 * z * (k2 * zz - k3 * xx - k3 * yy), -k6 * C33 * x * z, -k6 * C33 * y * z,
            C33 * (k6 * zz - k3 * xx - k3 * yy));
    s.basis(13, C34 * x * (k4 * zz - xx - yy), C34 * (k4 * zz - k3 * xx - yy), -k2 * C34 * x * y, k8 * C34 * x * z);
    s.basis(14, C35 * z * (xx - yy), k2 * C35 * x * z, -k2 * C35 * y * z, C35 * (xx - yy));
    s.basis(15, C36 * x * (xx - k3 * yy), C36 * (k3 * xx - k3 * yy), -k6 * C36 * x * y, k0);
}

// K4b. Uses K1's FP64 conic and opacity (conic_o) and its pre-clamp colour sign bits instead of
// re-deriving them; re-derives t, J, W-rotated J, Sigma3 and the rotation with K1's device code.
template <int DEG, bool OVERWRITE>
__global__ void __launch_bounds__(128, 4) k_backward_gaussians(const float* __restrict__ P, int n, int stride, int bc,
                                                            Pose pose, int W, int H,
                                                            const uint64_t* __restrict__ depth_key,
                                                            const double4* __restrict__ conic_o,
                                                            const Splat32* __restrict__ splat,
                                                            const float4* __restrict__ acc, float* __restrict__ G,
                                                            ScreenStats st) {
    pdl_begin();
    const int gid = blockIdx.x * blockDim.x + threadIdx.x;
    if (gid >= n) return;
    const Planes pl{bc};
    if (depth_key[gid] == ~0ull) {  // culled: zero gradient (gradients.cpp:82-86), nothing to add
        if (OVERWRITE)
            for (int q = 0; q < pl.count(); ++q) G[static_cast<size_t>(q) * stride + gid] = 0.0f;
        return;
    }
    if (OVERWRITE) {  // SH bands above the active degree carry no gradient (gradients.cpp:202-203)
        constexpr int active_n = (DEG + 1) * (DEG + 1);
        for (int q = pl.sh(active_n, 0); q < pl.sh(bc, 0); ++q) G[static_cast<size_t>(q) * stride + gid] = 0.0f;
    }

    // the geometry parameters are loaded up front (their latency overlaps the SH backward below)
    float lsf[3], qf[4];
#pragma unroll
    for (int k = 0; k < 3; ++k) lsf[k] = __ldg(P + static_cast<size_t>(pl.lscale(k)) * stride + gid);
#pragma unroll
    for (int k = 0; k < 4; ++k) qf[k] = __ldg(P + static_cast<size_t>(pl.rot(k)) * stride + gid);
    const float4 a0 = acc[3 * static_cast<size_t>(gid)];
    const float4 a1 = acc[3 * static_cast<size_t>(gid) + 1];
    const float4 a2 = acc[3 * static_cast<size_t>(gid) + 2];
    const double4 co = conic_o[gid];
    // K4a accumulated sum(dL/dpower * d) and sum(dL/dpower * d d^T); dpower/dp = Q d with the
    // FP64 conic (gradients.cpp:148-152), dpower/dconic = (d_x^2 / 2, d_x d_y, d_y^2 / 2)
    const double sdx = a1.x, sdy = a1.y;
    const double d_p[2] = {co.x * sdx + co.y * sdy, co.y * sdx + co.z * sdy};

    // screen-space gradient and densification statistics (gradients.cpp:180-183)
    const double ds0 = d_p[0] * W * 0.5, ds1 = d_p[1] * H * 0.5;
    st.d_screen[gid] = make_float2(static_cast<float>(ds0), static_cast<float>(ds1));
    st.norm_sum[gid] += sqrt(ds0 * ds0 + ds1 * ds1);
    st.hits[gid] += 1;

    // opacity through the sigmoid (gradients.cpp:186-187)
    const double o = co.w;
    put_grad<OVERWRITE>(G, stride, pl.opacity(), gid, static_cast<double>(a0.w) * o * (1.0 - o));

    // camera-space centre (camera.cpp:21-23)
    double m[3] = {load_param(P, stride, 0, gid), load_param(P, stride, 1, gid), load_param(P, stride, 2, gid)};
    double t[3], t_r;
    world_to_camera(pose, m, t, &t_r);

    // colour: SH coefficients and the view-direction path (gradients.cpp:190-209); the
    // pre-clamp sign gate (:197-200) comes from K1 (same basis, same summation order)
    double d_m_sh[3];
    {
        const uint32_t neg = __float_as_uint(splat[gid].pad);
        ShBack<float, OVERWRITE> sb{P, G, stride, gid, pl,
                  {(neg & 1u) ? 0.0f : a0.x, (neg & 2u) ? 0.0f : a0.y, (neg & 4u) ? 0.0f : a0.z},
                  {0.0f, 0.0f, 0.0f}};
        double dir[3];
        view_dir(pose, t, t_r, dir);
        const float dirf[3] = {static_cast<float>(dir[0]), static_cast<float>(dir[1]), static_cast<float>(dir[2])};
        sh_backward<DEG>(sb, dirf);
        const double sdd[3] = {sb.dd[0], sb.dd[1], sb.dd[2]};
        const double dd = dot3(dir, sdd);
        for (int c = 0; c < 3; ++c) d_m_sh[c] = (sdd[c] - dir[c] * dd) * (1.0 / t_r);
    }

    // mean path: dL/dt = J^T dL/dp (gradients.cpp:212-213)
    double jac[6], jg[18];
    jacobian_equirect_and_grad_fast(t, t_r, W, H, jac, jg);
    double d_t[3] = {jac[0] * d_p[0] + jac[3] * d_p[1], jac[1] * d_p[0] + jac[4] * d_p[1],
                     jac[2] * d_p[0] + jac[5] * d_p[1]};

    // covariance path (gradients.cpp:216-254)
    const double qa = co.x, qb = co.y, qc = co.z;
    const double da = 0.5 * static_cast<double>(a1.z), db = 0.5 * static_cast<double>(a1.w),
                 dc = 0.5 * static_cast<double>(a2.x);
    const double m00 = qa * da + qb * db, m01 = qa * db + qb * dc;
    const double m10 = qb * da + qc * db, m11 = qb * db + qc * dc;
    const double dva = -(m00 * qa + m01 * qb);
    const double dvb = -(m00 * qb + m01 * qc);
    const double dvc = -(m10 * qb + m11 * qc);
    double m23[6];
    m23_mul(jac, pose.R, m23);
    const double* m0 = m23;
    const double* m1 = m23 + 3;
    double dsig[9];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c)
            dsig[r * 3 + c] = dva * m0[r] * m0[c] + dvb * (m0[r] * m1[c] + m1[r] * m0[c]) + dvc * m1[r] * m1[c];
    double s[3], q[4], s3[9];
#pragma unroll
    for (int k = 0; k < 3; ++k) s[k] = exp(static_cast<double>(lsf[k]));
#pragma unroll
    for (int k = 0; k < 4; ++k) q[k] = static_cast<double>(qf[k]);
    // normalised once, by one reciprocal (a few ulp from the reference's divisions; the gradients'
    // tolerance allows it), for Sigma, the rotation and the normalisation's gradient below
    const double inv_n = 1.0 / qnorm(q);
    double qu[4];
    qu[0] = q[0] * inv_n; qu[1] = q[1] * inv_n; qu[2] = q[2] * inv_n; qu[3] = q[3] * inv_n;
    covariance3d_unit(qu, s, s3);
    double sm0[3], sm1[3];
    m3v(s3, m0, sm0);
    m3v(s3, m1, sm1);
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
#pragma unroll
    for (int r = 0; r < 6; ++r) {
        const double dj = djac[r];
        d_t[0] += jg[3 * r + 0] * dj;
        d_t[1] += jg[3 * r + 1] * dj;
        d_t[2] += jg[3 * r + 2] * dj;
    }
    double dpos[3];
    m3tv(pose.R, d_t, dpos);
    for (int c = 0; c < 3; ++c) put_grad<OVERWRITE>(G, stride, c, gid, dpos[c] + d_m_sh[c]);

    // Sigma3 -> quaternion (through normalisation) and log-scales (gradients.cpp:260-293)
    double rot[9];
    quat_rot(qu, rot);
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
    const double qdot = qu[0] * dqu[0] + qu[1] * dqu[1] + qu[2] * dqu[2] + qu[3] * dqu[3];
#pragma unroll
    for (int k = 0; k < 4; ++k) put_grad<OVERWRITE>(G, stride, pl.rot(k), gid, (dqu[k] - qu[k] * qdot) * inv_n);
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const double rk[3] = {rot[k], rot[3 + k], rot[6 + k]};
        double srk[3];
        m3v(dsig, rk, srk);
        const double rr = dot3(rk, srk);
        put_grad<OVERWRITE>(G, stride, pl.lscale(k), gid, 2.0 * s[k] * rr * s[k]);
    }
}



// ---- deterministic mode (optional) ----------------------------------------------
// K4a with a fixed summation order, the analogue of gradients.cpp:94-169 (per-tile accumulators,
// then a fixed-order reduction): the tile walks its list 64 entries at a time (staged by the first
// 64 threads, same records and masks as K4a); every quarter reduces an entry's 9 values over its 16
// pixels with the same shuffle tree as K4a and stores the result in its own shared slot
// part[quarter][entry]; after the round the 16 slots of every entry are summed in quarter order and
// stored — no atomics — at the instance's emission index. The per-pair math is K4a's, instruction
// for instruction (the pair classifier is shared through pair.cuh; the update below restates
// K4a's body), so deterministic gradients equal K4a's up to FP32 summation order.
constexpr int kDetChunk = 64;

template <bool BG>
__global__ void __launch_bounds__(kTileThreads) k_backward_pixels_det(
    const uint32_t* __restrict__ inst_gid, const uint2* __restrict__ ranges, PreprocessOut pp, int W, int H,
    int tiles_x, float bg0, float bg1, float bg2, FrameBuffers fb, const float* __restrict__ d_image,
    const uint32_t* __restrict__ inv_rank, const uint32_t* __restrict__ rank_off, const int2* __restrict__ rank_rc,
    float* __restrict__ inst_acc) {
    __shared__ WarpStage stage[kDetChunk / 32];
    __shared__ uint16_t s_mask[kDetChunk];
    __shared__ float part[2 * kTileWarps][kDetChunk][9];
    __shared__ int s_last[kTileWarps];
    const int tile = block_tile(tiles_x, (H + kTile - 1) / kTile);
    const int tx = tile % tiles_x, ty = tile / tiles_x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const WarpPixel wp = warp_pixel(warp, lane);
    const int lx = wp.lx, ly = wp.ly;
    const int px = tx * kTile + lx, py = ty * kTile + ly;
    const bool inside = px < W && py < H;
    const uint2 range = ranges[tile];
    const double width = W;
    const double xc = tx * kTile + 8.0, yc = ty * kTile + 8.0;
    const float lxo = lx - 7.5f, lyo = ly - 7.5f;
    const float halfW = 0.5f * W, fW = static_cast<float>(W);
    const float2 nlo = make_float2(-lxo, -lyo);
    const size_t pix = static_cast<size_t>(py) * W + px;
    const size_t plane = static_cast<size_t>(W) * H;
    const int last = inside ? fb.last[pix] : 0;
    const float T_final = inside ? fb.T[pix] : 0.0f;
    const float dl0 = inside ? d_image[pix] : 0.0f;
    const float dl1 = inside ? d_image[plane + pix] : 0.0f;
    const float2 dl01 = make_float2(dl0, dl1);
    const float dl2 = inside ? d_image[2 * plane + pix] : 0.0f;
    const float bg_dot = bg0 * dl0 + bg1 * dl1 + bg2 * dl2;
    const int max_last = static_cast<int>(__reduce_max_sync(0xffffffffu, static_cast<unsigned>(last)));
    const int quarter = 2 * warp + wp.half;
    float T_acc = T_final;
    float2 ns01 = make_float2(0.0f, 0.0f);
    float ns2 = 0.0f;
    if (lane == 0) s_last[warp] = max_last;
    __syncthreads();
    int cta_last = 0;
#pragma unroll
    for (int w = 0; w < kTileWarps; ++w) cta_last = max(cta_last, s_last[w]);
    const int t = threadIdx.x;
    float* partf = &part[0][0][0];
    for (int hi = cta_last; hi > 0; hi -= kDetChunk) {
        const int lo = hi > kDetChunk ? hi - kDetChunk : 0;
        for (int u = t; u < 2 * kTileWarps * kDetChunk * 9; u += kTileThreads) partf[u] = 0.0f;
        if (t < kDetChunk) {
            const int i = lo + t;
            uint32_t m = 0u;
            if (i < hi) {
                const uint32_t gid = inst_gid[range.x + i];
                const float4* s4 = reinterpret_cast<const float4*>(pp.splat + gid);
                m = stage_record16<true>(stage[t >> 5], t & 31, gid, pp.pxy[gid], s4[0], s4[1], s4[2], xc, yc, width);
            }
            s_mask[t] = static_cast<uint16_t>(m);
        }
        __syncthreads();
        for (int sub = kDetChunk / 32 - 1; sub >= 0; --sub) {
            const int sbase = lo + 32 * sub;
            if (sbase >= hi || sbase >= max_last) continue;
            const WarpStage& ws = stage[sub];
            const uint32_t mk = s_mask[32 * sub + lane];
            const uint32_t bal0 = __ballot_sync(0xffffffffu, (mk >> (2 * warp)) & 1u);
            const uint32_t bal1 = __ballot_sync(0xffffffffu, (mk >> (2 * warp + 1)) & 1u);
            uint32_t bal = wp.half ? bal1 : bal0;
            while (__any_sync(0xffffffffu, bal != 0u)) {
                const bool live = bal != 0u;
                const int j = live ? 31 - __clz(bal) : 0;
                bal &= ~(1u << j);
                const int k = sbase + j;
                float v[9] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
                bool has = false;
                if (live && k < last) {
                    const float4 A = ws.a[j];
                    const float4 B = ws.b[j];
                    float2 d;
                    float power;
                    bool unc;
                    if (pair_power2(A, B, nlo, halfW, fW, d, power, unc)) {
                        const float4 Cc = ws.c[j];
                        float alpha, g;
                        bool gate;
                        bool ok = true;
                        if (unc) {
                            Pair64 p;
                            ok = pair_slow(ws.gid[j], px, py, width, pp.pxy, pp.conic_o, &p);
                            alpha = static_cast<float>(p.alpha);
                            g = static_cast<float>(p.g);
                            gate = p.og < kAlphaMax;
                        } else {
                            g = ex2_approx(-power * kLog2e);
                            const float og = Cc.w * g;
                            alpha = fminf(0.99f, og);
                            gate = true;
                            if (Cc.w >= 0.98f) {
                                const float band = 0.99f * (1.5f * fabsf(B.w) + 1e-6f);
                                if (fabsf(og - 0.99f) <= band) {
                                    Pair64 p;
                                    pair_slow(ws.gid[j], px, py, width, pp.pxy, pp.conic_o, &p);
                                    gate = p.og < kAlphaMax;
                                } else {
                                    gate = og < 0.99f;
                                }
                            }
                        }
                        if (ok) {
                            has = true;
                            const float one_m = 1.0f - alpha;
                            float inv;
                            asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(inv) : "f"(one_m));
                            T_acc = T_acc * inv;
                            const float wb = alpha * T_acc;
                            const float2 v01 = __fmul2_rn(dl01, make_float2(wb, wb));
                            v[0] = v01.x;
                            v[1] = v01.y;
                            v[2] = dl2 * wb;
                            const float2 cs = __fadd2_rn(make_float2(Cc.x, Cc.y), ns01);
                            float d_alpha = cs.x * dl01.x;
                            d_alpha = __fmaf_rn(cs.y, dl01.y, d_alpha);
                            d_alpha = __fmaf_rn(Cc.z + ns2, dl2, d_alpha);
                            d_alpha = d_alpha * T_acc;
                            if (BG) d_alpha = d_alpha - (T_final * inv) * bg_dot;
                            const float nalpha = -alpha;
                            ns01 = __ffma2_rn(make_float2(Cc.x, Cc.y), make_float2(nalpha, nalpha),
                                              __fmul2_rn(ns01, make_float2(one_m, one_m)));
                            ns2 = __fmaf_rn(Cc.z, nalpha, ns2 * one_m);
                            if (gate) {
                                v[3] = g * d_alpha;
                                const float d_power = -Cc.w * v[3];
                                const float2 v45 = __fmul2_rn(d, make_float2(d_power, d_power));
                                const float2 v67 = __fmul2_rn(d, make_float2(v45.x, v45.x));
                                v[4] = v45.x;
                                v[5] = v45.y;
                                v[6] = v67.x;
                                v[7] = v67.y;
                                v[8] = v45.y * d.y;
                            }
                        }
                    }
                }
                const uint32_t hb_all = __ballot_sync(0xffffffffu, has);
                if (hb_all == 0u) continue;
                int idx;
                const float sum = half_reduce9(v, lane, &idx);
                // each quarter visits an entry at most once: its slot is written once per round
                const uint32_t hb = hb_all & (wp.half ? 0xFFFF0000u : 0x0000FFFFu);
                if (live && hb != 0u && idx >= 0) part[quarter][32 * sub + j][idx] = sum;
            }
            __syncwarp();
        }
        __syncthreads();
        // fixed-order combination over the 16 quarters, stored at the emission index
        for (int u = t; u < kDetChunk * 9; u += kTileThreads) {
            const int j = u / 9, i = u - 9 * j;
            if (lo + j >= hi) continue;
            float acc_v = 0.0f;
#pragma unroll
            for (int q = 0; q < 2 * kTileWarps; ++q) acc_v += part[q][j][i];
            const uint32_t gid = stage[j >> 5].gid[j & 31];
            const uint32_t r = inv_rank[gid];
            const int2 rc = rank_rc[r];
            const int x0 = static_cast<int>(static_cast<int16_t>(rc.x & 0xFFFF));
            const int wt = static_cast<int>(static_cast<uint32_t>(rc.x) >> 16);
            int col = tx - x0;
            col = ((col % tiles_x) + tiles_x) % tiles_x;
            const size_t e = static_cast<size_t>(rank_off[r]) + static_cast<size_t>(ty - rc.y) * wt + col;
            inst_acc[e * 9 + i] = acc_v;
        }
        __syncthreads();
    }
}

__global__ void k_inv_rank(const uint32_t* __restrict__ rank_gid, int n, uint32_t* __restrict__ inv_rank) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r < n) inv_rank[rank_gid[r]] = static_cast<uint32_t>(r);
}

// Pass 2: one thread per depth rank sums its instances in emission order (FP64) -> acc (FP32).
__global__ void k_det_reduce(const uint32_t* __restrict__ rank_off, const uint32_t* __restrict__ rank_gid,
                             const uint32_t* __restrict__ touched, int n, const float* __restrict__ inst_acc,
                             float4* __restrict__ acc) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    const uint32_t gid = rank_gid[r];
    const uint32_t cnt = touched[gid];
    if (cnt == 0u) return;
    double s[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    const float* p = inst_acc + static_cast<size_t>(rank_off[r]) * 9;
    for (uint32_t li = 0; li < cnt; ++li, p += 9)
#pragma unroll
        for (int i = 0; i < 9; ++i) s[i] += static_cast<double>(p[i]);
    float4* a = acc + 3 * static_cast<size_t>(gid);
    a[0] = make_float4(static_cast<float>(s[0]), static_cast<float>(s[1]), static_cast<float>(s[2]),
                       static_cast<float>(s[3]));
    a[1] = make_float4(static_cast<float>(s[4]), static_cast<float>(s[5]), static_cast<float>(s[6]),
                       static_cast<float>(s[7]));
    a[2] = make_float4(static_cast<float>(s[8]), 0.0f, 0.0f, 0.0f);
}

}  // namespace

void launch_backward_pixels_det(const uint32_t* inst_gid, const uint2* ranges, const PreprocessOut& pp, int W, int H,
                                int tiles_x, int tiles_y, const float bg[3], const FrameBuffers& fb,
                                const float* d_image, const EmitArrays& em, int n, uint32_t* inv_rank,
                                float* inst_acc, float4* acc, cudaStream_t s) {
    const int tiles = tiles_x * tiles_y;
    if (tiles <= 0 || n <= 0) return;
    k_inv_rank<<<(n + 255) / 256, 256, 0, s>>>(em.rank_gid, n, inv_rank);
    if (bg[0] != 0.0f || bg[1] != 0.0f || bg[2] != 0.0f)
        k_backward_pixels_det<true><<<tiles, kTileThreads, 0, s>>>(inst_gid, ranges, pp, W, H, tiles_x, bg[0], bg[1],
                                                                   bg[2], fb, d_image, inv_rank, em.rank_off,
                                                                   em.rank_rc, inst_acc);
    else
        k_backward_pixels_det<false><<<tiles, kTileThreads, 0, s>>>(inst_gid, ranges, pp, W, H, tiles_x, bg[0], bg[1],
                                                                    bg[2], fb, d_image, inv_rank, em.rank_off,
                                                                    em.rank_rc, inst_acc);
    k_det_reduce<<<(n + 255) / 256, 256, 0, s>>>(em.rank_off, em.rank_gid, pp.touched, n, inst_acc, acc);
    OSB_LAUNCHED(3);
}


#ifdef OSB_K4A_STATS
extern "C" __attribute__((visibility("default"))) void osb_k4a_stats(unsigned long long out[8], int reset) {
    cudaMemcpyFromSymbol(out, g_k4a_stats, sizeof(unsigned long long) * 8);
    if (reset) {
        unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        cudaMemcpyToSymbol(g_k4a_stats, z, sizeof(z));
    }
}
#endif

void launch_backward_pixels(const uint32_t* inst_gid, const uint2* ranges, const PreprocessOut& pp, int W, int H,
                            int tiles_x, int tiles_y, const float bg[3], const FrameBuffers& fb, const float* d_image,
                            float4* acc, cudaStream_t s) {
    const int tiles = tiles_x * tiles_y;
    if (tiles <= 0) return;
    if (bg[0] != 0.0f || bg[1] != 0.0f || bg[2] != 0.0f)
        launch_pdl(k_backward_pixels<true>, tiles, kTileThreads, s, inst_gid, ranges, pp, W, H, tiles_x, bg[0], bg[1],
                   bg[2], fb, d_image, acc);
    else
        launch_pdl(k_backward_pixels<false>, tiles, kTileThreads, s, inst_gid, ranges, pp, W, H, tiles_x, bg[0],
                   bg[1], bg[2], fb, d_image, acc);
    OSB_LAUNCHED(1);
}

void launch_backward_gaussians(const float* params, int n, int stride, int bc, int active_degree, const Pose& pose,
                               int W, int H, const PreprocessOut& pp, const float4* acc, float* grads,
                               const ScreenStats& st, bool overwrite, cudaStream_t s) {
    if (n <= 0) return;
    const int blocks = (n + 127) / 128;
#define OSB_K4B(D, O)                                                                                               \
    launch_pdl(k_backward_gaussians<D, O>, blocks, 128, s, params, n, stride, bc, pose, W, H, pp.depth_key,       \
               pp.conic_o, pp.splat, acc, grads, st)
    switch (active_degree * 2 + (overwrite ? 1 : 0)) {
        case 0: OSB_K4B(0, false); break;
        case 1: OSB_K4B(0, true); break;
        case 2: OSB_K4B(1, false); break;
        case 3: OSB_K4B(1, true); break;
        case 4: OSB_K4B(2, false); break;
        case 5: OSB_K4B(2, true); break;
        case 6: OSB_K4B(3, false); break;
        default: OSB_K4B(3, true); break;
    }
#undef OSB_K4B
    OSB_LAUNCHED(1);
}

}  // namespace osb
