// pair.cuh — the per-(pixel, splat) evaluation shared by K3 (blend) and K4a (backward pixels).
//
// Shared-memory staging record per tile-list entry (3 x float4, broadcast reads):
//   A = {cx, cy, ha, hc}   centre offset from the tile centre (FP64 -> FP32, seam-wrapped), 0.5 conic
//   B = {b, plo, phi, dl}  conic b, pthr -/+ delta, delta (negative: per-pixel seam wrap needed)
//   Cc = {r, g, bl, o}     colour, opacity
// The FP32 decision is "certain" outside the guard band and identical in K3 and K4a (same
// instructions, --fmad=false, explicit FMAs), so the backward replays the forward's decisions.
#pragma once

#include "common.cuh"

namespace osb {

constexpr int kStage = 256;
constexpr float kLog2e = 1.4426950408889634f;

struct StageSmem {
    float4 a[kStage];
    float4 b[kStage];
    float4 c[kStage];
    uint32_t gid[kStage];
};

// Stage tile-list entry `idx` (global instance index) into slot j.
__device__ __forceinline__ void stage_splat(StageSmem& sm, int j, uint32_t gid, const double2* __restrict__ pxy,
                                            const Splat32* __restrict__ splat, const float* __restrict__ delta,
                                            double xc, double yc, double width) {
    const double2 pp = pxy[gid];
    const Splat32 sp = splat[gid];
    const float dl = delta[gid];
    const double w0 = remainder(pp.x - xc, width);
    const bool seam = fabs(w0) > 0.5 * width - 8.5;
    sm.a[j] = make_float4(static_cast<float>(w0), static_cast<float>(pp.y - yc), sp.ha, sp.hc);
    sm.b[j] = make_float4(sp.b, sp.pthr - dl, sp.pthr + dl, seam ? -dl : dl);
    sm.c[j] = make_float4(sp.r, sp.g, sp.bl, sp.o);
    sm.gid[j] = gid;
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
static __device__ __noinline__ int pair_slow(uint32_t gid, int px, int py, double width, const double2* __restrict__ pxy,
                                      const double4* __restrict__ conic_o, Pair64* out) {
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
static __device__ __noinline__ double replay_T(const uint32_t* __restrict__ inst_gid, uint32_t lo, uint32_t k, int px,
                                        int py, double width, const double2* __restrict__ pxy,
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
