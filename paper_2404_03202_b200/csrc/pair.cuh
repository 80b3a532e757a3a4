// pair.cuh — the per-(pixel, splat) evaluation shared by K3 (blend) and K4a (backward pixels).
//
// Tile layout: one 256-thread CTA per 16x16 tile, one pixel per thread; warp w owns the 8x4 pixel
// block at columns 8(w&1)..+7, rows 4(w>>1)..+3, and each half-warp one 4x4 quarter of it (small
// square blocks are touched by far fewer splats than 16-pixel strips of the same area). The CTA
// walks its tile's list 512 entries at a time: every thread stages two entries into shared memory
// (stage_record16) with a 16-bit mask of the quarters its conservative alpha >= 1/255 extent
// (Splat32::ext_x/ext_y; in K4a further cut by per-row ellipse intervals) reaches; after one barrier every warp walks the staged entries, each
// half-warp only those whose bit for its quarter is set (ballots) — entries outside are certain
// skips of the FP32 classifier below, so no decision changes. K3 walks front to back and stops when
// every pixel has terminated; K4a walks back to front from each warp's furthest last_contrib.
//
// Staged record per entry (3 x float4, broadcast reads):
//   A = {cx, cy, ha, hc}   centre offset from the tile centre (FP64 -> FP32, seam-wrapped), 0.5 conic
//   B = {b, plo, phi, dl}  conic b, pthr -/+ delta, delta (negative: per-pixel seam wrap needed)
//   Cc = {r, g, bl, o}     colour, opacity
// The FP32 decision is "certain" outside the guard band and identical in K3 and K4a (same
// instructions, --fmad=false, explicit FMAs), so the backward replays the forward's decisions.
#pragma once

#include "common.cuh"

namespace osb {

constexpr int kTileThreads = 256;
constexpr int kTileWarps = kTileThreads / 32;
constexpr float kLog2e = 1.4426950408889634f;

// Pixel of (warp, lane) inside the tile, and the warp block's first row/column offset from the tile
// centre.
struct WarpPixel {
    int lx, ly, half;
    float r0, c0;
};
__device__ __forceinline__ WarpPixel warp_pixel(int warp, int lane) {
    WarpPixel w;
    w.half = lane >> 4;
    w.lx = (warp & 1) * 8 + w.half * 4 + (lane & 3);
    w.ly = (warp >> 1) * 4 + ((lane >> 2) & 3);
    w.r0 = static_cast<float>((warp >> 1) * 4) - 7.5f;
    w.c0 = static_cast<float>((warp & 1) * 8) - 7.5f;
    return w;
}

struct WarpStage {
    float4 a[32];
    float4 b[32];
    float4 c[32];
    uint32_t gid[32];
};

// Staged-record reads through a 32-bit shared-memory address computed (and pinned in a register)
// once per kernel: indexing stage[sub].a[j] directly makes the compiler rebuild the shared window
// base (S2R + LEA + 2 IMAD) on every iteration of the hot loops.
struct StageRef {
    uint32_t base;  // shared address of stage[sub]
    __device__ __forceinline__ float4 a(int j) const { return ld4(base + 16u * j); }
    __device__ __forceinline__ float4 b(int j) const { return ld4(base + 512u + 16u * j); }
    __device__ __forceinline__ float4 c(int j) const { return ld4(base + 1024u + 16u * j); }
    __device__ __forceinline__ uint32_t gid(int j) const {
        uint32_t v;
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(base + 1536u + 4u * j));
        return v;
    }
    static __device__ __forceinline__ float4 ld4(uint32_t addr) {
        float4 v;
        asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
        return v;
    }
};
__device__ __forceinline__ uint32_t pinned_smem_base(const void* p) {
    uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(p));
    asm volatile("mov.b32 %0, %0;" : "+r"(a));
    return a;
}

// Stage entry `gid` into this lane's slot for the tile centred at (xc, yc); returns a 2-bit mask:
// bit h set when the entry can reach a pixel centre of half-warp h's block (row offsets r0..r0+3,
// column offsets c0+4h..c0+4h+3).
// 16-bit reach mask of a staged entry for the 16 4x4 quarters of its tile (quarter q = 2 warp +
// half: columns 4 (2 (w & 1) + half) .. +3, rows 4 (w >> 1) .. +3), from the same conservative
// alpha extents as stage_record's two-bit masks: a clear bit is a certain skip for every pixel of
// that quarter.
__device__ __forceinline__ uint32_t quarter_mask(const float4 A, float ext_x, float ext_y, bool seam) {
    const float cx = A.x, cy = A.y;
    uint32_t rows = 0u, cols = 0u;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        const float r0 = 4.0f * r - 7.5f;
        rows |= (cy - ext_y <= r0 + 3.0f && cy + ext_y >= r0) ? (1u << r) : 0u;
    }
    if (seam) {
        cols = 0xFu;
    } else {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const float c0 = 4.0f * c - 7.5f;
            cols |= (cx - ext_x <= c0 + 3.0f && cx + ext_x >= c0) ? (1u << c) : 0u;
        }
    }
    // quarter q: warp row = q >> 2, column group = q & 3 (= 2 (w & 1) + half)
    uint32_t m = 0u;
#pragma unroll
    for (int r = 0; r < 4; ++r)
        if (rows & (1u << r)) m |= cols << (4 * r);
    return m;
}

// Tighter per-row columns: for quarter row r (pixel-centre offsets y in [4r - 7.5, 4r - 4.5]) the
// pixels of the ellipse {d : ha dx^2 + b dx dy + hc dy^2 <= P} (d = centre - pixel) lie at
// x = cx - dx with dx in dxc(dy) -/+ hw(dy), dxc = -b dy / (2 ha) linear in dy and
// hw = sqrt(4 ha P - (4 ha hc - b^2) dy^2) / (2 ha) largest at the dy of the band closest to 0.
// The union over the band is bounded by [cx - max dxc - max hw, cx - min dxc + max hw]; det4 is taken
// from below and the interval widened (relative 1e-3 + 0.05 px), so a cleared bit stays a certain
// skip of the FP32 classifier (P = the extents' pthr + 3 delta bound, as for ext_x / ext_y).
__device__ __forceinline__ uint32_t ellipse_row_cols(float cx, float cy, float ha, float b, float hc, float P, int r,
                                                     uint32_t cols_box) {
    const float y0 = 4.0f * r - 7.5f;
    const float dylo = cy - (y0 + 3.0f), dyhi = cy - y0;
    const float dys = fminf(fmaxf(0.0f, dylo), dyhi);
    const float det4 = fmaxf(4.0f * ha * hc - b * b - 1e-5f * (4.0f * ha * hc + b * b), 0.0f);
    const float q = 4.0f * ha * P - det4 * dys * dys;
    if (!(ha > 0.0f) || !(q >= 0.0f)) return ha > 0.0f ? 0u : cols_box;  // band misses / degenerate: keep box
    // MUFU approximations (relative error ~2^-22, far inside the 1e-3 relative slack below)
    float rha, sq;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rha) : "f"(ha));
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(sq) : "f"(q));
    const float inv2ha = 0.5f * rha;
    const float hw = sq * inv2ha;
    const float d1 = -b * dylo * inv2ha, d2 = -b * dyhi * inv2ha;
    const float slack = 1e-3f * (fabsf(cx) + fabsf(d1) + fabsf(d2) + hw) + 0.05f;
    const float xlo = cx - fmaxf(d1, d2) - hw - slack, xhi = cx - fminf(d1, d2) + hw + slack;
    uint32_t cols = 0u;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        const float c0 = 4.0f * c - 7.5f;
        cols |= (xlo <= c0 + 3.0f && xhi >= c0) ? (1u << c) : 0u;
    }
    return cols & cols_box;
}

__device__ __forceinline__ uint32_t quarter_mask_ellipse(float cx, float cy, float ha, float b, float hc, float P,
                                                         float ext_x, float ext_y, bool seam) {
    const uint32_t box = quarter_mask(make_float4(cx, cy, 0.0f, 0.0f), ext_x, ext_y, seam);
    if (seam || box == 0u) return box;
    uint32_t m = 0u;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        const uint32_t row = (box >> (4 * r)) & 0xFu;
        if (row) m |= ellipse_row_cols(cx, cy, ha, b, hc, P, r, row) << (4 * r);
    }
    return m;
}

// stage_record for the CTA-cooperative walk: returns the 16-quarter reach mask — the extents'
// bounding box (quarter_mask), or with kEllipse the per-row ellipse intervals inside it (K4a: its
// per-entry work is heavier than the extra staging math; K3 stages entries its pixels may never
// reach and stays with the box: measured K3 0.508 -> 0.519 ms, K4a 1.071 -> 1.055 ms with ellipses).
template <bool kEllipse>
__device__ __forceinline__ uint32_t stage_record16(WarpStage& ws, int lane, uint32_t gid, const double2 pp,
                                                   const float4 s0, const float4 s1, const float4 s2, double xc,
                                                   double yc, double width) {
    double w0 = pp.x - xc;
    const double half = 0.5 * width;
    if (w0 > half) w0 -= width;
    else if (w0 < -half) w0 += width;
    const bool seam = fabs(w0) > half - 8.5;
    const float cx = static_cast<float>(w0), cy = static_cast<float>(pp.y - yc);
    const float dl = s2.x;
    ws.a[lane] = make_float4(cx, cy, s0.x, s0.z);
    ws.b[lane] = make_float4(s0.y, s1.w - dl, s1.w + dl, seam ? -dl : dl);
    ws.c[lane] = make_float4(s1.x, s1.y, s1.z, s0.w);
    ws.gid[lane] = gid;
    if (!kEllipse) return quarter_mask(make_float4(cx, cy, 0.0f, 0.0f), s2.y, s2.z, seam);
    const float P = (s1.w + 3.0f * dl) * (1.0f + 2e-4f) + 2e-3f;  // K1's extents bound, widened for FP32
    return quarter_mask_ellipse(cx, cy, s0.x, s0.y, s0.z, fmaxf(P, 0.0f), s2.y, s2.z, seam);
}

// FP32 power for one pair (pixel centre offset (lxo, lyo) from the tile centre; nlo = (-lxo, -lyo)).
// Returns false for a certain skip; `unc` is set when the FP32 result is within the guard band of a
// threshold (power < 0, alpha < 1/255) or of the seam wrap tie. The paired operations issue as
// packed f32x2 instructions (FADD2 / FMUL2: half the issue slots, each half rounded exactly like the
// scalar op), and K3 and K4a run exactly this code, so the backward replays the forward's decisions.
// SEAM = false: the caller knows no staged entry straddles the seam (B.w >= 0), so the wrap is skipped.
template <bool SEAM = true>
__device__ __forceinline__ bool pair_power2(const float4 A, const float4 B, float2 nlo, float halfW, float fW,
                                            float2& d, float& power, bool& unc) {
    d = __fadd2_rn(make_float2(A.x, A.y), nlo);  // (A.x - lxo, A.y - lyo)
    unc = false;
    if (SEAM && B.w < 0.0f) {
        if (d.x > halfW) d.x -= fW;
        else if (d.x < -halfW) d.x += fW;
        unc = fabsf(fabsf(d.x) - halfW) < 0.01f;
    }
    const float2 q = __fmul2_rn(make_float2(A.z, A.w), d);  // (A.z dx, A.w dy)
    const float bdx = B.x * d.x;
    power = __fmaf_rn(q.x, d.x, __fmaf_rn(q.y, d.y, bdx * d.y));
    if (!(power <= B.z) && !unc) return false;
    const float dl = fabsf(B.w);
    unc = unc || power < dl || power > B.y;
    return true;
}

// Tile of this CTA (K3 / K4a: one CTA per 16x16 tile), row-major. OSB_TILE_ORDER 1 launches the
// tile rows from the two image edges inwards (rows 0, R-1, 1, R-2, ...) so the long pole-row lists
// do not form the grid's tail (a list-scheduling model predicted -8 % for pole-heavy views); measured
// slower — K3 0.558 -> 0.571 ms, pole-heavy 603 -> 581 FPS: the CTAs in flight then cover two bands
// of rows instead of one, and the neighbouring tiles' shared splat records hit in L2 less often.
#ifndef OSB_TILE_ORDER
#define OSB_TILE_ORDER 0
#endif
__device__ __forceinline__ int block_tile(int tiles_x, int tiles_y) {
    const int b = blockIdx.x;
    if (OSB_TILE_ORDER == 0) return b;
    const int ri = b / tiles_x, col = b - ri * tiles_x;
    const int row = (ri & 1) ? tiles_y - 1 - (ri >> 1) : (ri >> 1);
    return row * tiles_x + col;
}

// Per-CTA context of the out-of-line FP64 fallbacks (K3, K4a): they read the FP64 records and
// recompute their pixel from the thread index, so none of it stays live in the hot loops' registers.
struct SlowCtx {
    const double2* pxy;
    const double4* conic_o;
    double width;
    int tiles_x;
    int tile;
};
static __shared__ SlowCtx s_slow;

__device__ __forceinline__ void slow_pixel(int& px, int& py) {
    const int tile = s_slow.tile;
    const WarpPixel wp = warp_pixel(threadIdx.x >> 5, threadIdx.x & 31);
    px = (tile % s_slow.tiles_x) * kTile + wp.lx;
    py = (tile / s_slow.tiles_x) * kTile + wp.ly;
}

__device__ __forceinline__ uint32_t bfind_u32(uint32_t x) {  // index of the highest set bit, ~0u for 0
    uint32_t r;
    asm("bfind.u32 %0, %1;" : "=r"(r) : "r"(x));
    return r;
}
__device__ __forceinline__ uint32_t below_u32(uint32_t j) {  // (1 << j) - 1, all ones for j >= 32 (one BMSK)
    uint32_t r;
    asm("bmsk.clamp.b32 %0, 0, %1;" : "=r"(r) : "r"(j));
    return r;
}
__device__ __forceinline__ uint32_t bit_u32(uint32_t j) {  // 1 << j, 0 for j >= 32 (PTX clamps the shift)
    uint32_t r;
    asm("shl.b32 %0, 1, %1;" : "=r"(r) : "r"(j));
    return r;
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

// replay_T done by the whole warp for one pixel (px, py): lane l evaluates entries lo + 32 r + l in
// FP64, then the factors are multiplied into t in list order (t * 1.0 == t for skipped entries,
// so the product equals the sequential reference loop bit for bit). All lanes must call it
// together; every lane returns the same t.
__device__ __forceinline__ double warp_replay_T(const uint32_t* __restrict__ inst_gid, uint32_t lo, uint32_t k,
                                                int px, int py, double width, const double2* __restrict__ pxy,
                                                const double4* __restrict__ conic_o, int lane) {
    double t = 1.0;
    const double sx = px + 0.5, sy = py + 0.5;
    for (uint32_t base = lo; base < k; base += 32) {
        const uint32_t i = base + lane;
        double f = 1.0;
        if (i < k) {
            const uint32_t g = __ldg(inst_gid + i);
            const double2 pc = pxy[g];
            const double4 co = conic_o[g];
            double gg, a;
            if (pair_fp64(pc.x, pc.y, co.x, co.y, co.z, co.w, sx, sy, width, &gg, &a)) f = 1.0 - a;
        }
        const int cnt = k - base < 32u ? static_cast<int>(k - base) : 32;
        for (int q = 0; q < cnt; ++q) t = t * __shfl_sync(0xffffffffu, f, q);
    }
    return t;
}

}  // namespace osb
