// pair.cuh — the per-(pixel, splat) evaluation shared by K3 (blend) and K4a (backward pixels).
//
// Shared-memory staging record per tile-list entry (3 x float4, broadcast reads):
//   A = {cx, cy, ha, hc}   centre offset from the tile centre (FP64 -> FP32, seam-wrapped), 0.5 conic
//   B = {b, plo, phi, dl}  conic b, pthr -/+ delta, delta (negative: per-pixel seam wrap needed)
//   Cc = {r, g, bl, o}     colour, opacity
// plus a warp mask: the 16x16 tile is 8 warps x 2 pixel rows; bit w is set when the entry's
// conservative extent (Splat32::ext_x/ext_y) reaches a pixel centre of warp w. Entries outside are
// certain skips in the FP32 classifier below, so dropping them per warp changes no decision.
// The FP32 decision is "certain" outside the guard band and identical in K3 and K4a (same
// instructions, --fmad=false, explicit FMAs), so the backward replays the forward's decisions.
#pragma once

#include "common.cuh"

namespace osb {

constexpr int kStage = 256;
constexpr int kStageWarps = kStage / 32;
constexpr float kLog2e = 1.4426950408889634f;

struct StageSmem {
    float4 a[kStage];
    float4 b[kStage];
    float4 c[kStage];
    uint32_t gid[kStage];
    uint8_t mask[kStage];
    uint8_t list[kStageWarps][kStage];  // per-warp compacted entry indices
};

// Stage entry j (Gaussian gid) for the tile centred at (xc, yc).
__device__ __forceinline__ void stage_splat(StageSmem& sm, int j, uint32_t gid, const double2* __restrict__ pxy,
                                            const Splat32* __restrict__ splat, double xc, double yc,
                                            double width) {
    const double2 pp = pxy[gid];
    const float4* s4 = reinterpret_cast<const float4*>(splat + gid);
    const float4 s0 = s4[0], s1 = s4[1], s2 = s4[2];  // {ha,b,hc,o} {r,g,bl,pthr} {dl,ext_x,ext_y,-}
    const double w0 = remainder(pp.x - xc, width);
    const bool seam = fabs(w0) > 0.5 * width - 8.5;
    const float cx = static_cast<float>(w0), cy = static_cast<float>(pp.y - yc);
    const float dl = s2.x;
    sm.a[j] = make_float4(cx, cy, s0.x, s0.z);
    sm.b[j] = make_float4(s0.y, s1.w - dl, s1.w + dl, seam ? -dl : dl);
    sm.c[j] = make_float4(s1.x, s1.y, s1.z, s0.w);
    sm.gid[j] = gid;
    uint32_t m = 0;
    if (seam || fabsf(cx) <= 7.5f + s2.y) {
        // pixel rows r (centre offset r - 7.5) with |cy - (r - 7.5)| <= ext_y
        const float lo = cy - s2.z + 7.5f, hi = cy + s2.z + 7.5f;
        const int rlo = lo <= 0.0f ? 0 : (lo > 15.0f ? 16 : static_cast<int>(ceilf(lo)));
        const int rhi = hi >= 15.0f ? 15 : (hi < 0.0f ? -1 : static_cast<int>(floorf(hi)));
        if (rlo <= rhi) m = ((2u << (rhi >> 1)) - 1u) & ~((1u << (rlo >> 1)) - 1u);
    }
    sm.mask[j] = static_cast<uint8_t>(m);
}

// Warp `warp` gathers the indices of the staged entries it can reach; returns how many.
__device__ __forceinline__ int compact_for_warp(StageSmem& sm, int cnt, int warp, int lane) {
    int n = 0;
    const uint32_t lt = lanemask_lt();
    for (int base = 0; base < cnt; base += 32) {
        const int e = base + lane;
        const bool act = e < cnt && ((sm.mask[e] >> warp) & 1u);
        const uint32_t bal = __ballot_sync(0xffffffffu, act);
        if (act) sm.list[warp][n + __popc(bal & lt)] = static_cast<uint8_t>(e);
        n += __popc(bal);
    }
    __syncwarp();
    return n;
}

// FP32 power for one pair. Returns false for a certain skip. `unc` is set when the FP32 result
// is within the guard band of a threshold (power < 0, alpha < 1/255) or of the seam wrap tie.
__device__ __forceinline__ bool pair_power(const float4 A, const float4 B, float lxo, float lyo, float halfW,
                                           float fW, float& dx, float& dy, float& power, bool& unc) {
    dx = A.x - lxo;
    dy = A.y - lyo;
    unc = false;
    if (B.w < 0.0f) {
        if (dx > halfW) dx -= fW;
        else if (dx < -halfW) dx += fW;
        unc = fabsf(fabsf(dx) - halfW) < 0.01f;
    }
    const float bdx = B.x * dx;
    power = __fmaf_rn(A.z * dx, dx, __fmaf_rn(A.w * dy, dy, bdx * dy));
    if (!(power <= B.z) && !unc) return false;
    const float dl = fabsf(B.w);
    unc = unc || power < dl || power > B.y;
    return true;
}

struct Pair64 {
    double alpha, g, og;
};

// Exact FP64 evaluation of instance `gid` at pixel (px, py) — rasterizer.cpp:128-134.
static __device__ __noinline__ int pair_slow(uint32_t gid, int px, int py, double width,
                                             const double2* __restrict__ pxy, const double4* __restrict__ conic_o,
                                             Pair64* out) {
    const double2 pp = pxy[gid];
    const double4 co = conic_o[gid];
    double g, alpha;
    if (!pair_fp64(pp.x, pp.y, co.x, co.y, co.z, co.w, px + 0.5, py + 0.5, width, &g, &alpha)) return 0;
    out->alpha = alpha;
    out->g = g;
    out->og = co.w * g;
    return 1;
}

// FP64 transmittance in front of list position `k` (exclusive), replaying the reference blend
// (rasterizer.cpp:126-141) over list[lo, k).
static __device__ __noinline__ double replay_T(const uint32_t* __restrict__ inst_gid, uint32_t lo, uint32_t k,
                                               int px, int py, double width, const double2* __restrict__ pxy,
                                               const double4* __restrict__ conic_o) {
    double t = 1.0;
    for (uint32_t i = lo; i < k; ++i) {
        Pair64 p;
        if (!pair_slow(inst_gid[i], px, py, width, pxy, conic_o, &p)) continue;
        t = t * (1.0 - p.alpha);
    }
    return t;
}

}  // namespace osb
