// sort.cu — K2: depth-rank sort, instance duplication, stable tile sort, tile ranges.
//
// Replaces bin_to_tiles (proj/src/rasterizer.cpp:57-98): the serial duplication loop and the
// per-tile std::sort by (depth, gaussian_id). Exactness argument:
//   1. all Gaussians are stably radix-sorted by the 64-bit pattern of t_r (positive doubles order
//      like their bit patterns; culled ones carry ~0 and sink to the end), with ids as values in
//      ascending order -> (depth, id) order;
//   2. instances are emitted in that order (exclusive scan of tiles_touched over it, then a
//      load-balanced emission: every lane writes consecutive instances -> coalesced stores);
//   3. a STABLE radix sort by tile id keeps the (depth, id) order inside every tile; its last pass
//      writes the per-tile ranges instead of the sorted keys.
// So each tile list equals the reference's sorted list element for element. The fast depth rank
// sorts 24-bit FP32-derived keys instead and restores the exact (FP64 depth, id) order inside runs
// of equal keys on the way into the emission (k_touch_sums).
//
// Radix sort: LSD, 8-bit digits, reduce-then-scan per digit (no serial cross-block chain — at these
// sizes every block is resident at once, so a decoupled look-back would serialise):
//   upsweep   per-block digit counts (warp-private shared histograms)
//   scan      per digit, exclusive prefix over blocks + the digit's global base
//   downsweep stable per-warp ranking (one ballot per digit bit), block-local sort in shared
//             memory, coalesced scatter of runs of equal digits.
// No host synchronization inside a sort.
#include "kernels.h"

namespace osb {

int scan_block_count(int n);

namespace {

constexpr int kRadixBits = 8;
constexpr int kBins = 1 << kRadixBits;
constexpr int kSortThreads = 256;
constexpr int kSortWarps = kSortThreads / 32;
constexpr int kMaxPasses = 8;

template <typename K>
struct SortCfg;
template <>
struct SortCfg<uint64_t> {
    static constexpr int kItems = 8;
};
template <>
struct SortCfg<uint32_t> {
    static constexpr int kItems = 8;
};
template <typename K>
__host__ __device__ constexpr int tile_keys() {
    return kSortThreads * SortCfg<K>::kItems;
}

// First pass of a sort may read its keys through a transform and take identity values:
// key24 != nullptr: the 24-bit depth key (bits - min) >> shift of K1's FP32 depth bits (culled:
// 0xFFFFFF), the range {min, ~max} of the visible bits at key24[0..1]; vals_in == nullptr: value =
// element index (the depth rank sorts Gaussian ids 0..n-1).
struct Key24 {
    uint32_t lo = 0;
    int shift = 0;
    bool on = false;
    __device__ explicit Key24(const uint32_t* range) {
        if (!range) return;
        on = true;
        lo = range[0];
        const uint32_t hi = ~range[1];
        const uint32_t span = hi >= lo ? hi - lo : 0u;
        while ((span >> shift) >= 0xFFFFFFu) ++shift;
    }
    template <typename K>
    __device__ __forceinline__ K operator()(K b) const {
        if (!on) return b;
        const uint32_t u = static_cast<uint32_t>(b);
        return static_cast<K>(u == 0xFFFFFFFFu ? 0xFFFFFFu : (u - lo) >> shift);
    }
};

// Element count of a sort: the host bound, or min(bound, *n_dev) when the count lives on the device
// (the tile sort runs before the host knows M; the grid is sized for the buffer capacity).
__device__ __forceinline__ int sort_count(int n_cap, const uint32_t* n_dev) {
    if (!n_dev) return n_cap;
    const uint32_t m = *n_dev;
    return m < static_cast<uint32_t>(n_cap) ? static_cast<int>(m) : n_cap;
}

// 256-thread exclusive scan (returns exclusive prefix, *total = block sum).
__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t v, uint32_t* s_warp, uint32_t* total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t inc = v;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, inc, off);
        if (lane >= off) inc += t;
    }
    if (lane == 31) s_warp[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        const uint32_t w = lane < kSortWarps ? s_warp[lane] : 0u;
        uint32_t wi = w;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, wi, off);
            if (lane >= off) wi += t;
        }
        if (lane < kSortWarps) s_warp[lane] = wi - w;
        if (lane == kSortWarps - 1) s_warp[kSortWarps] = wi;
    }
    __syncthreads();
    const uint32_t r = s_warp[warp] + inc - v;
    *total = s_warp[kSortWarps];
    return r;
}

// Per-block digit counts for one pass: counts[d * nblocks + b]. The first pass (hist != nullptr)
// also accumulates every pass's global digit totals hist[p][d] (one read of the keys serves both).
template <typename K>
__global__ void __launch_bounds__(kSortThreads) k_upsweep(const K* __restrict__ keys, int n_cap, const uint32_t* n_dev,
                                                          int shift, int nblocks, uint32_t* __restrict__ counts,
                                                          int passes, uint32_t* __restrict__ hist,
                                                          const uint32_t* __restrict__ key24) {
    pdl_begin();
    const int n = sort_count(n_cap, n_dev);
    const Key24 xf(key24);
    constexpr int kTile = tile_keys<K>();
    __shared__ uint32_t s_hist[kSortWarps][kBins];
    __shared__ uint32_t s_tot[kMaxPasses][kBins];
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < kSortWarps * kBins; i += kSortThreads) (&s_hist[0][0])[i] = 0;
    if (hist)
        for (int i = threadIdx.x; i < kMaxPasses * kBins; i += kSortThreads) (&s_tot[0][0])[i] = 0;
    __syncthreads();
    const long base = static_cast<long>(blockIdx.x) * kTile;
    const int count = static_cast<int>(max(0L, min(static_cast<long>(kTile), static_cast<long>(n) - base)));
    for (int i = threadIdx.x; i < count; i += kSortThreads) {
        const K k = xf(keys[base + i]);
        atomicAdd(&s_hist[warp][static_cast<uint32_t>((k >> shift) & (kBins - 1))], 1u);
        if (hist)
            for (int p = 1; p < passes; ++p)
                atomicAdd(&s_tot[p][static_cast<uint32_t>((k >> (p * kRadixBits)) & (kBins - 1))], 1u);
    }
    __syncthreads();
    uint32_t c = 0;
#pragma unroll
    for (int w = 0; w < kSortWarps; ++w) c += s_hist[w][threadIdx.x];
    counts[static_cast<size_t>(threadIdx.x) * nblocks + blockIdx.x] = c;
    if (hist) {
        if (c) atomicAdd(&hist[threadIdx.x], c);
        for (int p = 1; p < passes; ++p) {
            const uint32_t t = s_tot[p][threadIdx.x];
            if (t) atomicAdd(&hist[p * kBins + threadIdx.x], t);
        }
    }
}

// One block per digit: offsets[d][b] = digit_base[d] + sum_{b' < b} counts[d][b'], the digit base
// being the exclusive prefix of this pass's global digit totals.
__global__ void __launch_bounds__(kSortThreads) k_scan_counts(const uint32_t* __restrict__ counts, int nblocks,
                                                              const uint32_t* __restrict__ digit_totals,
                                                              uint32_t* __restrict__ offsets) {
    pdl_begin();
    __shared__ uint32_t s_scan[kSortWarps + 1];
    __shared__ uint32_t s_base;
    const int d = blockIdx.x;
    {
        uint32_t total;
        const uint32_t ex = block_exclusive_scan(digit_totals[threadIdx.x], s_scan, &total);
        if (static_cast<int>(threadIdx.x) == d) s_base = ex;
        __syncthreads();  // s_base visible; s_scan free for the next scan
    }
    // each thread sums a contiguous run of blocks, one block-wide scan, then the run is written
    const uint32_t* row = counts + static_cast<size_t>(d) * nblocks;
    uint32_t* out = offsets + static_cast<size_t>(d) * nblocks;
    const int per = (nblocks + kSortThreads - 1) / kSortThreads;
    const int b0 = threadIdx.x * per, b1 = min(b0 + per, nblocks);
    uint32_t local = 0;
    for (int b = b0; b < b1; ++b) local += row[b];
    uint32_t total;
    uint32_t run = s_base + block_exclusive_scan(local, s_scan, &total);
    for (int b = b0; b < b1; ++b) {
        const uint32_t v = row[b];
        out[b] = run;
        run += v;
    }
}

template <typename K>
__global__ void __launch_bounds__(kSortThreads) k_downsweep(const K* __restrict__ keys_in,
                                                            const uint32_t* __restrict__ vals_in,
                                                            K* __restrict__ keys_out, uint32_t* __restrict__ vals_out,
                                                            int n_cap, const uint32_t* n_dev, int shift, int nblocks,
                                                            const uint32_t* __restrict__ offsets,
                                                            const uint32_t* __restrict__ key24,
                                                            uint2* __restrict__ ranges) {
    pdl_begin();
    const int n = sort_count(n_cap, n_dev);
    const Key24 xf(key24);
    if (static_cast<long>(blockIdx.x) * kSortThreads * SortCfg<K>::kItems >= n) return;
    // this thread's digit offset (thread = digit), loaded with the keys instead of after the ranking
    const uint32_t my_off = offsets[static_cast<size_t>(threadIdx.x) * nblocks + blockIdx.x];
    constexpr int kItems = SortCfg<K>::kItems;
    constexpr int kTile = kSortThreads * kItems;
    __shared__ uint32_t s_warp[kSortWarps][kBins];
    __shared__ uint32_t s_local[kBins];  // block-local start of each digit
    __shared__ int s_global[kBins];      // global position - local position, per digit
    __shared__ uint32_t s_scan[kSortWarps + 1];
    __shared__ K s_keys[kTile];
    __shared__ uint32_t s_vals[kTile];

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int i = tid; i < kSortWarps * kBins; i += kSortThreads) (&s_warp[0][0])[i] = 0;
    __syncthreads();
    const uint32_t bid = blockIdx.x;
    const long block_base = static_cast<long>(bid) * kTile;
    const long base = block_base + static_cast<long>(warp) * 32 * kItems;
    const int count = static_cast<int>(min(static_cast<long>(kTile), static_cast<long>(n) - block_base));

    K key[kItems];
    uint32_t val[kItems];
    uint16_t rank[kItems];
    const uint32_t lt = lanemask_lt();
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
        const long idx = base + i * 32 + lane;
        const bool valid = idx < n;
        key[i] = valid ? xf(keys_in[idx]) : K(0);
        val[i] = valid ? (vals_in ? vals_in[idx] : static_cast<uint32_t>(idx)) : 0u;
    }
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
        const long idx = base + i * 32 + lane;
        const bool valid = idx < n;
        const uint32_t d = valid ? static_cast<uint32_t>((key[i] >> shift) & (kBins - 1)) : kBins;
        // lanes with the same digit: one ballot per digit bit (match.any has a long latency here)
        uint32_t peers = __ballot_sync(0xffffffffu, valid);
#pragma unroll
        for (int b = 0; b < kRadixBits; ++b) {
            const bool bit = (d >> b) & 1u;
            const uint32_t vote = __ballot_sync(0xffffffffu, bit);
            peers &= bit ? vote : ~vote;
        }
        if (!valid) peers = 1u << lane;
        const int leader = __ffs(peers) - 1;
        uint32_t prev = 0;
        if (valid && lane == leader) {
            prev = s_warp[warp][d];
            s_warp[warp][d] = prev + __popc(peers);
        }
        prev = __shfl_sync(0xffffffffu, prev, leader);
        rank[i] = static_cast<uint16_t>(prev + __popc(peers & lt));
        __syncwarp();
    }
    __syncthreads();

    // Per digit (thread = digit): exclusive prefix over warps and the block count.
    const int d = tid;
    uint32_t cnt = 0;
#pragma unroll
    for (int w = 0; w < kSortWarps; ++w) {
        const uint32_t t = s_warp[w][d];
        s_warp[w][d] = cnt;
        cnt += t;
    }
    uint32_t total;
    const uint32_t local = block_exclusive_scan(cnt, s_scan, &total);
    s_local[d] = local;
    s_global[d] = static_cast<int>(my_off) - static_cast<int>(local);
    __syncthreads();

    // Block-local sort into shared memory.
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
        const long idx = base + i * 32 + lane;
        if (idx < n) {
            const uint32_t dd = static_cast<uint32_t>((key[i] >> shift) & (kBins - 1));
            const uint32_t pos = s_local[dd] + s_warp[warp][dd] + rank[i];
            s_keys[pos] = key[i];
            s_vals[pos] = val[i];
        }
    }
    __syncthreads();
    // Coalesced scatter: consecutive local positions of one digit are consecutive globally.
    if (!ranges) {
        for (int i = tid; i < count; i += kSortThreads) {
            const K k = s_keys[i];
            const uint32_t dd = static_cast<uint32_t>((k >> shift) & (kBins - 1));
            const int dst = s_global[dd] + i;
            keys_out[dst] = k;
            vals_out[dst] = s_vals[i];
        }
        return;
    }
    // Last pass of the tile sort: the sorted keys are only needed for the tile ranges, so they are
    // not stored; the ranges come from here. Inside this block's run of one digit the keys are in
    // final (tile) order and consecutive globally, so a tile boundary between two neighbours of the
    // run is a plain store; at the run's two ends the global neighbour belongs to another block, so
    // the start / end are combined with atomicMin / atomicMax (ranges start at {~0u, 0}: K1 or k_k2_zero;
    // the one plain store of a boundary is the extremum, so the order against the atomics is free).
    for (int i = tid; i < count; i += kSortThreads) {
        const uint32_t k = static_cast<uint32_t>(s_keys[i]);
        const uint32_t dd = (k >> shift) & (kBins - 1);
        const int lo = static_cast<int>(s_local[dd]);
        const int hi = dd + 1 < kBins ? static_cast<int>(s_local[dd + 1]) : count;  // run of digit dd: [lo, hi)
        const int dst = s_global[dd] + i;
        vals_out[dst] = s_vals[i];
        if (i == lo) atomicMin(&ranges[k].x, static_cast<uint32_t>(dst));
        else if (static_cast<uint32_t>(s_keys[i - 1]) != k) ranges[k].x = static_cast<uint32_t>(dst);
        if (i == hi - 1) atomicMax(&ranges[k].y, static_cast<uint32_t>(dst + 1));
        else if (static_cast<uint32_t>(s_keys[i + 1]) != k) ranges[k].y = static_cast<uint32_t>(dst + 1);
    }
}

// ---- scan of tiles_touched (depth order) + load-balanced instance emission ----------------------
constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;  // ranks per block

constexpr int kMaxRun = 64;

// Exact (FP64 depth, id) order inside a run of equal FP32-rounded depth keys around rank r (the
// stable FP32 sort left the run in ascending id order): the rank this element takes inside the run,
// or -1 when the run is longer than kMaxRun (*flag raised: the caller redoes the depth rank with
// the full 64-bit sort). O(run length) per member, every member places itself.
__device__ __noinline__ int run_position(const uint32_t* __restrict__ keys, const uint32_t* __restrict__ order,
                                         const uint64_t* __restrict__ depth_key, int n, int r, uint32_t k,
                                         uint32_t g, uint32_t* flag) {
    int s = r, e = r + 1;
    while (s > 0 && keys[s - 1] == k && r - s < kMaxRun) --s;
    while (e < n && keys[e] == k && e - r <= kMaxRun) ++e;
    if (e - s > kMaxRun) {
        atomicExch(flag, 1u);
        return -1;
    }
    const uint64_t d = depth_key[g];
    int below = 0;
    for (int a = s; a < e; ++a) {
        const uint32_t h = order[a];
        const uint64_t dh = depth_key[h];
        below += (dh < d || (dh == d && h < g)) ? 1 : 0;
    }
    return s + below;
}

// Per depth rank r: the Gaussian that takes rank r (rank_gid), its touched count (rank_off, read
// by k_emit_prep) and packed tile rectangle {x0 & 0xFFFF | width << 16, y0} (rank_rc; both gathers
// issued together), and the per-block sums of touched (atomics into sums zeroed by K1 or k_k2_zero).
// keys (fast depth rank): the sorted 24-bit keys; every element of a run of equal keys places itself
// at its exact (FP64 depth, id) position inside the run (replaces a separate run-fixing pass; a run
// may straddle two blocks, so its elements add to the sum of the block they land in).
__global__ void __launch_bounds__(kScanThreads) k_touch_sums(const uint32_t* __restrict__ touched,
                                                             const uint32_t* __restrict__ order, int n,
                                                             uint32_t* __restrict__ block_sums,
                                                             uint32_t* __restrict__ ranked,
                                                             uint32_t* __restrict__ rank_gid,
                                                             const int4* __restrict__ rect,
                                                             int2* __restrict__ rank_rc,
                                                             const uint32_t* __restrict__ keys,
                                                             const uint64_t* __restrict__ depth_key,
                                                             uint32_t* __restrict__ flag) {
    pdl_begin();
    __shared__ uint32_t s_scan[kSortWarps + 1];
    const long r0 = static_cast<long>(blockIdx.x) * kScanTile + threadIdx.x;
    uint32_t local = 0;
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
        const long r = r0 + i * kScanThreads;
        if (r < n) {
            const uint32_t g = order[r];
            long dst = r;
            if (keys) {
                const uint32_t k = keys[r];
                if (k != 0xFFFFFFu && ((r > 0 && keys[r - 1] == k) || (r + 1 < n && keys[r + 1] == k))) {
                    const int p = run_position(keys, order, depth_key, n, static_cast<int>(r), k, g, flag);
                    if (p >= 0) dst = p;
                }
            }
            const uint32_t v = touched[g];
            const int4 q = rect[g];  // stale for culled Gaussians (v = 0): not used then
            ranked[dst] = v;
            rank_gid[dst] = g;
            rank_rc[dst] = v > 0 ? make_int2((q.x & 0xFFFF) | ((q.y - q.x + 1) << 16), q.z) : make_int2(0, 0);
            if (dst / kScanTile == blockIdx.x) local += v;
            else if (v) atomicAdd(&block_sums[dst / kScanTile], v);
        }
    }
    uint32_t total;
    block_exclusive_scan(local, s_scan, &total);
    if (threadIdx.x == 0 && total) atomicAdd(&block_sums[blockIdx.x], total);
}

// Instance emission in depth order, balanced over OUTPUTS (the instance counts per rank are very
// skewed: full-width pole splats emit hundreds of tiles): k_emit_prep writes, per depth rank, its
// first output (exclusive scan), id and packed tile rectangle; k_emit gives every CTA exactly
// kEmitTile consecutive outputs, finds the ranks covering them with two global binary searches,
// stages their first-outputs in shared memory, and every thread emits 8 consecutive instances (one
// shared-memory search, then a forward walk). Stores are 32-B runs per lane.
constexpr int kEmitTile = kScanThreads * 8;
constexpr int kEmitWindow = 2 * kEmitTile;  // ranks staged per CTA (more only with many empty ranks)
constexpr int kEmitSmall = kEmitWindow / 4;  // windows up to this also stage their gid / rectangle records
static_assert(4 * kEmitSmall * 4 <= kEmitWindow * 4, "off + gid + rc fit in the s_off space");

// rank_off[r] holds the touched count of rank r on entry (k_touch_sums) and the rank's first output
// on exit. Each block derives its own exclusive prefix from the raw block sums (at most a few
// thousand words: cheaper than a separate scan launch); the last block stores M = *total.
__global__ void __launch_bounds__(kScanThreads) k_emit_prep(int n, const uint32_t* __restrict__ block_sums,
                                                            uint32_t* __restrict__ rank_off,
                                                            uint32_t* __restrict__ total,
                                                            uint32_t* __restrict__ cta_first, int nctas) {
    pdl_begin();
    __shared__ uint32_t s_scan[kSortWarps + 1];
    const long r0 = static_cast<long>(blockIdx.x) * kScanTile + threadIdx.x * kScanItems;
    uint32_t v[kScanItems];
    uint32_t local = 0;
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
        const long r = r0 + i;
        v[i] = r < n ? rank_off[r] : 0u;
        local += v[i];
    }
    uint32_t before = 0;
    for (int b = threadIdx.x; b < static_cast<int>(blockIdx.x); b += kScanThreads) before += block_sums[b];
    uint32_t agg, base_all;
    block_exclusive_scan(before, s_scan, &base_all);
    __syncthreads();  // s_scan is reused
    uint32_t run = base_all + block_exclusive_scan(local, s_scan, &agg);
    if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) *total = base_all + agg;
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
        const long r = r0 + i;
        if (r >= n) break;
        rank_off[r] = run;
        // the rank owning output b * kEmitTile starts k_emit's CTA b (no binary search there);
        // entry nctas bounds the last CTA's window when M exceeds the capacity
        if (v[i] > 0 && cta_first)
            for (uint32_t b = (run + kEmitTile - 1) / kEmitTile; b <= (run + v[i] - 1) / kEmitTile &&
                                                                  b <= static_cast<uint32_t>(nctas); ++b)
                cta_first[b] = static_cast<uint32_t>(r);
        run += v[i];
    }
}

// last index e in [0, count) with off[e] <= o (off non-decreasing, off[0] <= o)
__device__ __forceinline__ int owner_of(const uint32_t* off, int count, uint32_t o) {
    int lo = 0, hi = count - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (off[mid] <= o) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

// The emitted instances are staged in shared memory and written with 16-byte stores; with `counts`
// the CTA also produces the tile sort's first-pass upsweep for its block (sort block b = emission
// CTA b: both cover 2048 consecutive instances): the low-digit counts of its keys at counts[d *
// nblocks + b] and both passes' global digit totals in hist (the tile sort then skips that upsweep).
__global__ void __launch_bounds__(kScanThreads) k_emit(const uint32_t* __restrict__ rank_off,
                                                       const uint32_t* __restrict__ rank_gid,
                                                       const int2* __restrict__ rank_rc, int n,
                                                       const uint32_t* __restrict__ total, int tiles_x,
                                                       uint32_t* __restrict__ keys, uint32_t* __restrict__ vals,
                                                       uint32_t capacity, const uint32_t* __restrict__ cta_first,
                                                       uint32_t* __restrict__ counts, uint32_t* __restrict__ hist,
                                                       int nblocks) {
    pdl_begin();
    __shared__ __align__(16) uint32_t s_off[kEmitWindow];
    __shared__ __align__(16) uint32_t s_k[kEmitTile];
    __shared__ __align__(16) uint32_t s_v[kEmitTile];
    __shared__ uint32_t s_h0[kBins], s_h1[kBins];
    __shared__ int s_rb, s_w;
    const uint32_t M = *total;
    const uint32_t o_begin = static_cast<uint32_t>(blockIdx.x) * kEmitTile;
    if (o_begin >= M) {
        if (counts) counts[static_cast<size_t>(threadIdx.x) * nblocks + blockIdx.x] = 0u;
        return;
    }
    const uint32_t o_end = min(o_begin + static_cast<uint32_t>(kEmitTile), M);
    if (counts) {
        s_h0[threadIdx.x] = 0u;
        s_h1[threadIdx.x] = 0u;
    }
    if (threadIdx.x == 0) {
        // first rank from k_emit_prep; the owner of the next CTA's first output bounds the window
        // (the last CTA searches: the culled ranks with no instances follow it)
        const int rb = static_cast<int>(cta_first[blockIdx.x]);
        const int re = o_end < M ? static_cast<int>(cta_first[blockIdx.x + 1])
                                 : rb + owner_of(rank_off + rb, n - rb, o_end - 1);
        s_rb = rb;
        s_w = re - rb + 1;
    }
    __syncthreads();
    const int rb = s_rb, w = s_w;
    const uint32_t* off = rank_off + rb;
    const uint32_t* gidp = rank_gid + rb;
    const int2* rcp = rank_rc + rb;
    if (w <= kEmitSmall) {
        // the window's whole records in shared memory (one coalesced load phase instead of a
        // dependent global load at every rank change of the walk): off | gid | rc in s_off's space
        uint32_t* s_gid = s_off + kEmitSmall;
        int2* s_rc = reinterpret_cast<int2*>(s_off + 2 * kEmitSmall);
        for (int i = threadIdx.x; i < w; i += kScanThreads) {
            s_off[i] = off[i];
            s_gid[i] = gidp[i];
            s_rc[i] = rcp[i];
        }
        __syncthreads();
        off = s_off;
        gidp = s_gid;
        rcp = s_rc;
    } else if (w <= kEmitWindow) {
        for (int i = threadIdx.x; i < w; i += kScanThreads) s_off[i] = off[i];
        __syncthreads();
        off = s_off;
    }
    uint32_t o = o_begin + threadIdx.x * 8;
    if (o < o_end) {
        int e = owner_of(off, w, o);
        // the rank's record and the (row, column) of output o inside its rectangle: one division for
        // the thread's first output, then stepped along the row-major walk; reloaded when the rank changes
        int2 rc = rcp[e];
        uint32_t gid = gidp[e];
        uint32_t wt = static_cast<uint32_t>(rc.x) >> 16;
        uint32_t li = o - off[e];
        uint32_t row = li / wt, col = li - row * wt;
        uint32_t next = e + 1 < w ? off[e + 1] : 0xFFFFFFFFu;
        for (int q = 0; q < 8 && o < o_end; ++q, ++o) {
            if (o >= next) {  // o belongs to a later rank (skip ranks without instances)
                do {
                    ++e;
                    next = e + 1 < w ? off[e + 1] : 0xFFFFFFFFu;
                } while (o >= next);
                rc = rcp[e];
                gid = gidp[e];
                wt = static_cast<uint32_t>(rc.x) >> 16;
                row = 0;
                col = 0;
            }
            const int x0 = static_cast<int>(static_cast<int16_t>(rc.x & 0xFFFF));
            int kx = x0 + static_cast<int>(col);
            kx = kx < 0 ? kx + tiles_x : (kx >= tiles_x ? kx - tiles_x : kx);
            const uint32_t key = static_cast<uint32_t>((rc.y + static_cast<int>(row)) * tiles_x + kx);
            s_k[o - o_begin] = key;
            s_v[o - o_begin] = gid;
            if (counts && o < capacity) {
                atomicAdd(&s_h0[key & (kBins - 1)], 1u);
                atomicAdd(&s_h1[(key >> kRadixBits) & (kBins - 1)], 1u);
            }
            if (++col == wt) {
                col = 0;
                ++row;
            }
        }
    }
    __syncthreads();
    const uint32_t cnt = min(o_end, capacity) > o_begin ? min(o_end, capacity) - o_begin : 0u;
    if (cnt == static_cast<uint32_t>(kEmitTile)) {  // full block: 16-byte stores
        for (int i = threadIdx.x; i < kEmitTile / 4; i += kScanThreads) {
            reinterpret_cast<uint4*>(keys + o_begin)[i] = reinterpret_cast<const uint4*>(s_k)[i];
            reinterpret_cast<uint4*>(vals + o_begin)[i] = reinterpret_cast<const uint4*>(s_v)[i];
        }
    } else {
        for (uint32_t i = threadIdx.x; i < cnt; i += kScanThreads) {
            keys[o_begin + i] = s_k[i];
            vals[o_begin + i] = s_v[i];
        }
    }
    if (counts) {
        const uint32_t c0 = s_h0[threadIdx.x], c1 = s_h1[threadIdx.x];
        counts[static_cast<size_t>(threadIdx.x) * nblocks + blockIdx.x] = c0;
        if (c0) atomicAdd(&hist[threadIdx.x], c0);
        if (c1) atomicAdd(&hist[kBins + threadIdx.x], c1);
    }
}

// Tile ranges from stored sorted keys — only for a one-instance "sort" now (the tile sort's last
// downsweep writes the ranges otherwise). Four keys per thread (one 16-byte load + the two
// neighbours): a range starts where the key differs from its predecessor, ends where it differs from
// its successor.
__global__ void __launch_bounds__(256) k_ranges(const uint32_t* __restrict__ keys, int m_cap, const uint32_t* m_dev,
                                                uint2* __restrict__ ranges) {
    pdl_begin();
    const int m = sort_count(m_cap, m_dev);
    const int i0 = 4 * (blockIdx.x * blockDim.x + threadIdx.x);
    if (i0 >= m) return;
    uint32_t k[6];  // keys[i0 - 1 .. i0 + 4]
    if (i0 + 4 <= m) {
        const uint4 v = *reinterpret_cast<const uint4*>(keys + i0);
        k[1] = v.x; k[2] = v.y; k[3] = v.z; k[4] = v.w;
    } else {
#pragma unroll
        for (int q = 0; q < 4; ++q) k[1 + q] = i0 + q < m ? keys[i0 + q] : 0xFFFFFFFFu;
    }
    k[0] = i0 > 0 ? keys[i0 - 1] : 0xFFFFFFFFu;
    k[5] = i0 + 4 < m ? keys[i0 + 4] : 0xFFFFFFFFu;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int i = i0 + q;
        if (i >= m) break;
        const uint32_t c = k[1 + q];
        if (i == 0 || k[q] != c) ranges[c].x = i;
        if (i == m - 1 || k[2 + q] != c) ranges[c].y = i + 1;
    }
}

// Workspace: hist[8][256] (global digit totals per pass) | unused[8][256] | counts[256][blocks] |
// offsets[256][blocks]
template <typename K>
bool radix_sort(const K* first_keys, const uint32_t* key24, K* keys_in, K* keys_out, const uint32_t* first_vals,
                uint32_t* vals_in, uint32_t* vals_out, int n, const uint32_t* n_dev, int bits, void* ws,
                cudaStream_t s, bool counts_ready = false, int hist_slot = 0, bool hist_zeroed = false,
                uint2* ranges = nullptr) {
    if (n <= 1) {
        if (n == 1 && !first_vals) OSB_CUDA_CHECK(cudaMemsetAsync(vals_in, 0, sizeof(uint32_t), s));  // id 0
        if (ranges && n == 1)
            launch_pdl(k_ranges, 1, 256, s, reinterpret_cast<const uint32_t*>(keys_in), n, n_dev, ranges);
        return false;
    }
    const int passes = (bits + kRadixBits - 1) / kRadixBits;
    const int blocks = (n + tile_keys<K>() - 1) / tile_keys<K>();
    // workspace: two digit-total slots hist[2][kMaxPasses][kBins] (depth rank: 0, tile sort: 1, so
    // k_k2_zero can clear both before either runs) | counts[kBins][blocks] | offsets[kBins][blocks]
    uint32_t* hist = static_cast<uint32_t*>(ws) + hist_slot * kMaxPasses * kBins;
    uint32_t* counts = static_cast<uint32_t*>(ws) + 2 * kMaxPasses * kBins;
    uint32_t* offsets = counts + static_cast<size_t>(kBins) * blocks;
    if (!counts_ready && !hist_zeroed)
        OSB_CUDA_CHECK(cudaMemsetAsync(hist, 0, sizeof(uint32_t) * kMaxPasses * kBins, s));
    bool flipped = false;
    for (int p = 0; p < passes; ++p) {
        const K* ki = p == 0 ? first_keys : (flipped ? keys_out : keys_in);
        K* ko = flipped ? keys_in : keys_out;
        const uint32_t* vi = p == 0 ? first_vals : (flipped ? vals_out : vals_in);
        uint32_t* vo = flipped ? vals_in : vals_out;
        const uint32_t* xf = p == 0 ? key24 : nullptr;
        const int shift = p * kRadixBits;
        if (!(p == 0 && counts_ready)) {
            launch_pdl(k_upsweep<K>, blocks, kSortThreads, s, ki, n, n_dev, shift, blocks, counts, passes,
                       p == 0 ? hist : nullptr, xf);
            OSB_LAUNCHED(1);
        }
        launch_pdl(k_scan_counts, kBins, kSortThreads, s, counts, blocks, hist + p * kBins, offsets);
        launch_pdl(k_downsweep<K>, blocks, kSortThreads, s, ki, vi, ko, vo, n, n_dev, shift, blocks, offsets, xf,
                   p == passes - 1 ? ranges : nullptr);
        OSB_LAUNCHED(2);
        flipped = !flipped;
    }
    return flipped;
}

}  // namespace

size_t radix_workspace_bytes(int n_max, int key_bytes) {
    (void)key_bytes;  // sized for the smaller tile of either key type (the buffer serves both sorts)
    const int tk = tile_keys<uint64_t>() < tile_keys<uint32_t>() ? tile_keys<uint64_t>() : tile_keys<uint32_t>();
    const size_t blocks = (static_cast<size_t>(n_max) + tk - 1) / tk;
    return sizeof(uint32_t) * (2 * kMaxPasses * kBins + 2 * kBins * blocks) + 256;
}

bool radix_sort_u64(uint64_t* ki, uint64_t* ko, uint32_t* vi, uint32_t* vo, int n, int bits, void* ws,
                    cudaStream_t s, const uint64_t* first_keys, bool iota_vals, bool hist_zeroed) {
    return radix_sort<uint64_t>(first_keys ? first_keys : ki, nullptr, ki, ko, iota_vals ? nullptr : vi, vi, vo, n,
                                nullptr, bits, ws, s, false, 0, hist_zeroed);
}
bool radix_sort_u32(uint32_t* ki, uint32_t* ko, uint32_t* vi, uint32_t* vo, int n, int bits, void* ws,
                    cudaStream_t s, const uint32_t* n_dev, bool counts_ready, bool tile_slot, uint2* ranges) {
    return radix_sort<uint32_t>(ki, nullptr, ki, ko, vi, vi, vo, n, n_dev, bits, ws, s, counts_ready && bits <= 16,
                                tile_slot ? 1 : 0, tile_slot, ranges);
}
void tile_sort_prepare(void* ws, cudaStream_t s) {
    OSB_CUDA_CHECK(cudaMemsetAsync(static_cast<uint32_t*>(ws) + kMaxPasses * kBins, 0,
                                   sizeof(uint32_t) * kMaxPasses * kBins, s));
}
bool radix_sort_depth24(const uint32_t* depth_bits, const uint32_t* range, uint32_t* ki, uint32_t* ko, uint32_t* vi,
                        uint32_t* vo, int n, void* ws, cudaStream_t s, bool hist_zeroed) {
    return radix_sort<uint32_t>(depth_bits, range, ki, ko, nullptr, vi, vo, n, nullptr, 24, ws, s, false, 0,
                                hist_zeroed);
}

namespace {
// The frame's K2 scratch that must start at zero, in one chained kernel instead of separate memsets:
// both digit-total slots of the sort workspace, the long-run flag and the tile ranges.
__global__ void k_k2_zero(uint32_t* __restrict__ hist, int nhist, uint32_t* __restrict__ flag,
                          uint2* __restrict__ ranges, int tiles, uint32_t* __restrict__ scan_sums, int nsums) {
    pdl_begin();
    const int i = blockIdx.x * blockDim.x + threadIdx.x, step = gridDim.x * blockDim.x;
    for (int k = i; k < nhist; k += step) hist[k] = 0u;
    for (int k = i; k < nsums; k += step) scan_sums[k] = 0u;
    for (int k = i; k < tiles; k += step) ranges[k] = make_uint2(~0u, 0u);  // atomicMin / atomicMax identities
    if (i == 0) *flag = 0u;
}
}  // namespace

K2Scratch k2_scratch(void* sort_ws, uint32_t* long_run_flag, uint2* ranges, int tiles, void* scan_ws, int n) {
    K2Scratch z;
    z.hist = static_cast<uint32_t*>(sort_ws);
    z.nhist = 2 * kMaxPasses * kBins;
    z.flag = long_run_flag;
    z.ranges = ranges;
    z.tiles = tiles;
    z.sums = static_cast<uint32_t*>(scan_ws);
    z.nsums = scan_block_count(n);
    return z;
}

void launch_k2_zero(void* sort_ws, uint32_t* long_run_flag, uint2* ranges, int tiles, void* scan_ws, int n,
                    cudaStream_t s) {
    launch_pdl(k_k2_zero, 64, 256, s, static_cast<uint32_t*>(sort_ws), 2 * kMaxPasses * kBins, long_run_flag, ranges,
               tiles, static_cast<uint32_t*>(scan_ws), scan_block_count(n));
    OSB_LAUNCHED(1);
}

long emit_ctas(uint32_t capacity) { return (static_cast<long>(capacity) + kEmitTile - 1) / kEmitTile; }

size_t scan_workspace_bytes(int n) {
    const size_t blocks = (static_cast<size_t>(n) + kScanTile - 1) / kScanTile;
    return sizeof(uint32_t) * (blocks + 128) + (static_cast<size_t>(n) + 64) * 16 + 256;
}

EmitArrays scan_emit_arrays(void* ws, int n) {
    const int blocks = (n + kScanTile - 1) / kScanTile;
    uint32_t* sums = static_cast<uint32_t*>(ws);
    EmitArrays a;
    uint32_t* rank_off = sums + ((blocks + 64 + 63) & ~63);
    const size_t npad = (static_cast<size_t>(n) + 63) & ~size_t(63);
    a.rank_off = rank_off;
    a.rank_gid = rank_off + npad;
    a.rank_rc = reinterpret_cast<const int2*>(rank_off + 2 * npad);
    return a;
}

void launch_scan_emit(const uint32_t* touched, const uint32_t* order, const int4* rect, int n, int tiles_x,
                      uint32_t* keys, uint32_t* vals, uint32_t capacity, uint32_t* total, void* ws,
                      uint32_t* cta_first, void* tile_sort_ws, cudaStream_t s, const uint32_t* depth_keys24,
                      const uint64_t* depth_key, uint32_t* long_run_flag) {
    if (n <= 0) {
        OSB_CUDA_CHECK(cudaMemsetAsync(total, 0, sizeof(uint32_t), s));
        return;
    }
    const int blocks = (n + kScanTile - 1) / kScanTile;
    uint32_t* sums = static_cast<uint32_t*>(ws);  // zeroed by k_k2_zero (scan_sums_reset after a counting pass)
    uint32_t* rank_off = sums + ((blocks + 64 + 63) & ~63);
    const size_t npad = (static_cast<size_t>(n) + 63) & ~size_t(63);  // keeps every array 256-B aligned
    uint32_t* rank_gid = rank_off + npad;
    int2* rank_rc = reinterpret_cast<int2*>(rank_gid + npad);
    launch_pdl(k_touch_sums, blocks, kScanThreads, s, touched, order, n, sums, rank_off, rank_gid, rect, rank_rc,
               depth_keys24, depth_key, long_run_flag);
    // one CTA per kEmitTile outputs up to the capacity (CTAs past M exit; M > capacity is retried)
    const long grid = keys ? emit_ctas(capacity) : 0;
    launch_pdl(k_emit_prep, blocks, kScanThreads, s, n, sums, rank_off, total, cta_first, static_cast<int>(grid));
    // the tile sort's workspace layout (radix_sort): hist[kMaxPasses][kBins] | .. | counts[kBins][blocks]
    uint32_t* t_hist = tile_sort_ws ? static_cast<uint32_t*>(tile_sort_ws) + kMaxPasses * kBins : nullptr;  // slot 1
    uint32_t* t_counts = tile_sort_ws ? static_cast<uint32_t*>(tile_sort_ws) + 2 * kMaxPasses * kBins : nullptr;
    static_assert(kEmitTile == kSortThreads * SortCfg<uint32_t>::kItems, "emission CTA = tile-sort block");
    if (grid > 0)
        launch_pdl(k_emit, static_cast<int>(grid), kScanThreads, s, rank_off, rank_gid, rank_rc, n, total, tiles_x,
                   keys, vals, capacity, cta_first, t_counts, t_hist, static_cast<int>(grid));
    OSB_LAUNCHED(grid > 0 ? 3 : 2);
}

int scan_block_count(int n) { return n > 0 ? (n + kScanTile - 1) / kScanTile : 0; }

void scan_sums_reset(void* ws, int n, cudaStream_t s) {
    const int blocks = scan_block_count(n);
    if (blocks) OSB_CUDA_CHECK(cudaMemsetAsync(ws, 0, sizeof(uint32_t) * blocks, s));
}

}  // namespace osb
