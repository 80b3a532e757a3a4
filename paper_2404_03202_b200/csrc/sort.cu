// sort.cu — K2: depth-rank sort, instance duplication, stable tile sort, tile ranges.
//
// Replaces bin_to_tiles (proj/src/rasterizer.cpp:57-98): the serial duplication loop and the
// per-tile std::sort by (depth, gaussian_id). Exactness argument:
//   1. visible Gaussians are stably radix-sorted by the 64-bit pattern of t_r (positive doubles
//      order like their bit patterns), with ids as values in ascending order -> (depth, id) order;
//   2. instances are emitted in that order (exclusive scan of tiles_touched over it);
//   3. a STABLE radix sort by tile id keeps the (depth, id) order inside every tile.
// So each tile list equals the reference's sorted list element for element.
//
// Radix sort: LSD, 8-bit digits, one "onesweep" kernel per digit: per-warp match_any ranking,
// per-block digit counts, decoupled look-back across blocks for the global digit offsets
// (dynamic block ids guarantee forward progress). Digits that are constant over all keys are
// skipped (their counts are known from the up-front histogram).
#include <vector>

#include "kernels.h"

namespace osb {

namespace {

constexpr int kRadixBits = 8;
constexpr int kBins = 1 << kRadixBits;
constexpr int kSortThreads = 256;
constexpr int kSortWarps = kSortThreads / 32;
constexpr int kItems = 16;
constexpr int kTileKeys = kSortThreads * kItems;
constexpr uint32_t kFlagAgg = 1u << 30;
constexpr uint32_t kFlagPrefix = 2u << 30;
constexpr uint32_t kCountMask = (1u << 30) - 1;

template <typename K>
__global__ void __launch_bounds__(256) k_histogram(const K* __restrict__ keys, int n, int passes,
                                                   uint32_t* __restrict__ hist /* passes x 256 */) {
    __shared__ uint32_t s_hist[8][kBins];
    for (int i = threadIdx.x; i < passes * kBins; i += blockDim.x) (&s_hist[0][0])[i] = 0;
    __syncthreads();
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        K k = keys[i];
        for (int p = 0; p < passes; ++p) atomicAdd(&s_hist[p][(k >> (p * kRadixBits)) & (kBins - 1)], 1u);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < passes * kBins; i += blockDim.x) {
        uint32_t v = (&s_hist[0][0])[i];
        if (v) atomicAdd(&hist[i], v);
    }
}

// Exclusive scan of each pass's 256 digit counts -> digit base offsets. One block per pass.
__global__ void k_scan_hist(const uint32_t* __restrict__ hist, uint32_t* __restrict__ base) {
    __shared__ uint32_t s[kBins];
    const int p = blockIdx.x;
    const int d = threadIdx.x;
    s[d] = hist[p * kBins + d];
    __syncthreads();
    for (int off = 1; off < kBins; off <<= 1) {
        uint32_t v = d >= off ? s[d - off] : 0;
        __syncthreads();
        s[d] += v;
        __syncthreads();
    }
    base[p * kBins + d] = s[d] - hist[p * kBins + d];
}

template <typename K>
__global__ void __launch_bounds__(kSortThreads) k_onesweep(const K* __restrict__ keys_in,
                                                           const uint32_t* __restrict__ vals_in,
                                                           K* __restrict__ keys_out, uint32_t* __restrict__ vals_out,
                                                           int n, int shift, const uint32_t* __restrict__ digit_base,
                                                           uint32_t* __restrict__ status, uint32_t* __restrict__ counter) {
    __shared__ uint32_t s_bid;
    __shared__ uint32_t s_warp[kSortWarps][kBins];
    __shared__ uint32_t s_prefix[kBins];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) s_bid = atomicAdd(counter, 1u);
    for (int i = tid; i < kSortWarps * kBins; i += kSortThreads) (&s_warp[0][0])[i] = 0;
    __syncthreads();
    const uint32_t bid = s_bid;
    const long base = static_cast<long>(bid) * kTileKeys + static_cast<long>(warp) * 32 * kItems;

    K key[kItems];
    uint32_t val[kItems];
    uint32_t rank[kItems];
    const uint32_t lt = lanemask_lt();
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
        const long idx = base + i * 32 + lane;
        const bool valid = idx < n;
        key[i] = valid ? keys_in[idx] : K(0);
        val[i] = valid ? vals_in[idx] : 0u;
        const uint32_t d = valid ? static_cast<uint32_t>((key[i] >> shift) & (kBins - 1)) : kBins;
        const uint32_t peers = __match_any_sync(0xffffffffu, d);
        const int leader = __ffs(peers) - 1;
        uint32_t prev = 0;
        if (valid && lane == leader) {
            prev = s_warp[warp][d];
            s_warp[warp][d] = prev + __popc(peers);
        }
        prev = __shfl_sync(0xffffffffu, prev, leader);
        rank[i] = prev + __popc(peers & lt);
        __syncwarp();
    }
    __syncthreads();

    // Per digit: exclusive prefix over warps, block total, then look-back across blocks.
    {
        const int d = tid;
        uint32_t sum = 0;
#pragma unroll
        for (int w = 0; w < kSortWarps; ++w) {
            uint32_t t = s_warp[w][d];
            s_warp[w][d] = sum;
            sum += t;
        }
        uint32_t* my = status + static_cast<size_t>(bid) * kBins + d;
        uint32_t exclusive = 0;
        if (bid == 0) {
            st_release(my, kFlagPrefix | sum);
        } else {
            st_release(my, kFlagAgg | sum);
            long p = static_cast<long>(bid) - 1;
            while (true) {
                uint32_t s = ld_acquire(status + static_cast<size_t>(p) * kBins + d);
                uint32_t flag = s & ~kCountMask;
                if (flag == 0) continue;
                exclusive += s & kCountMask;
                if (flag == kFlagPrefix) break;
                --p;
            }
            st_release(my, kFlagPrefix | (exclusive + sum));
        }
        s_prefix[d] = digit_base[d] + exclusive;
    }
    __syncthreads();

#pragma unroll
    for (int i = 0; i < kItems; ++i) {
        const long idx = base + i * 32 + lane;
        if (idx < n) {
            const uint32_t d = static_cast<uint32_t>((key[i] >> shift) & (kBins - 1));
            const uint32_t dst = s_prefix[d] + s_warp[warp][d] + rank[i];
            keys_out[dst] = key[i];
            vals_out[dst] = val[i];
        }
    }
}

__global__ void k_iota(uint32_t* v, int n) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) v[i] = static_cast<uint32_t>(i);
}

// Single-pass exclusive scan with decoupled look-back over touched[order[r]].
constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;

__global__ void __launch_bounds__(kScanThreads) k_gather_scan(const uint32_t* __restrict__ touched,
                                                              const uint32_t* __restrict__ order,
                                                              uint32_t* __restrict__ out, uint32_t* __restrict__ total,
                                                              int n, uint32_t* __restrict__ status,
                                                              uint32_t* __restrict__ counter) {
    __shared__ uint32_t s_bid;
    __shared__ uint32_t s_warp[kScanThreads / 32];
    __shared__ uint32_t s_excl;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) s_bid = atomicAdd(counter, 1u);
    __syncthreads();
    const uint32_t bid = s_bid;
    const long base = static_cast<long>(bid) * kScanTile + static_cast<long>(tid) * kScanItems;
    uint32_t v[kScanItems];
    uint32_t local = 0;
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
        long idx = base + i;
        v[i] = idx < n ? touched[order[idx]] : 0u;
        local += v[i];
    }
    // block exclusive scan of per-thread sums
    uint32_t inc = local;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        uint32_t t = __shfl_up_sync(0xffffffffu, inc, off);
        if (lane >= off) inc += t;
    }
    if (lane == 31) s_warp[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        uint32_t w = lane < kScanThreads / 32 ? s_warp[lane] : 0u;
        uint32_t wi = w;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            uint32_t t = __shfl_up_sync(0xffffffffu, wi, off);
            if (lane >= off) wi += t;
        }
        if (lane < kScanThreads / 32) s_warp[lane] = wi - w;
        if (lane == kScanThreads / 32 - 1) {
            // block aggregate = wi (inclusive of the last warp); look back
            const uint32_t agg = wi;
            uint32_t excl = 0;
            if (bid == 0) {
                st_release(status + bid, kFlagPrefix | agg);
            } else {
                st_release(status + bid, kFlagAgg | agg);
                long p = static_cast<long>(bid) - 1;
                while (true) {
                    uint32_t s = ld_acquire(status + p);
                    uint32_t flag = s & ~kCountMask;
                    if (flag == 0) continue;
                    excl += s & kCountMask;
                    if (flag == kFlagPrefix) break;
                    --p;
                }
                st_release(status + bid, kFlagPrefix | (excl + agg));
            }
            s_excl = excl;
            if (static_cast<long>(bid + 1) * kScanTile >= n) *total = excl + agg;
        }
    }
    __syncthreads();
    uint32_t run = s_excl + s_warp[warp] + (inc - local);
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
        long idx = base + i;
        if (idx < n) out[idx] = run;
        run += v[i];
    }
}

// One thread per depth-sorted Gaussian: writes (tile, gid) for every tile of its rectangle.
__global__ void __launch_bounds__(256) k_emit(const uint32_t* __restrict__ order, const uint32_t* __restrict__ offsets,
                                              const uint32_t* __restrict__ touched, const int4* __restrict__ rect,
                                              int n, int tiles_x, uint32_t* __restrict__ keys,
                                              uint32_t* __restrict__ vals) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    const uint32_t gid = order[r];
    const uint32_t cnt = touched[gid];
    if (cnt == 0) return;
    const int4 rc = rect[gid];
    uint32_t o = offsets[r];
    for (int ty = rc.z; ty <= rc.w; ++ty)
        for (int k = rc.x; k <= rc.y; ++k) {
            int tx = ((k % tiles_x) + tiles_x) % tiles_x;
            keys[o] = static_cast<uint32_t>(ty * tiles_x + tx);
            vals[o] = gid;
            ++o;
        }
}

__global__ void k_ranges(const uint32_t* __restrict__ keys, int m, uint2* __restrict__ ranges) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    const uint32_t k = keys[i];
    if (i == 0 || keys[i - 1] != k) ranges[k].x = i;
    if (i == m - 1 || keys[i + 1] != k) ranges[k].y = i + 1;
}

struct RadixWs {
    uint32_t* hist;     // 8 x 256
    uint32_t* base;     // 8 x 256
    uint32_t* counter;  // 8
    uint32_t* status;   // 8 x blocks x 256
};

RadixWs carve(void* ws, int n_max) {
    const int blocks = (n_max + kTileKeys - 1) / kTileKeys;
    uint32_t* p = static_cast<uint32_t*>(ws);
    RadixWs r;
    r.hist = p;
    r.base = p + 8 * kBins;
    r.counter = p + 16 * kBins;
    r.status = p + 16 * kBins + 64;
    (void)blocks;
    return r;
}

template <typename K>
bool radix_sort(K* keys_in, K* keys_out, uint32_t* vals_in, uint32_t* vals_out, int n, int bits, void* ws,
                cudaStream_t s) {
    if (n <= 1) return false;
    const int passes = (bits + kRadixBits - 1) / kRadixBits;
    const int blocks = (n + kTileKeys - 1) / kTileKeys;
    RadixWs w = carve(ws, n);
    const size_t status_words = static_cast<size_t>(passes) * blocks * kBins;
    OSB_CUDA_CHECK(cudaMemsetAsync(w.hist, 0, sizeof(uint32_t) * (16 * kBins + 64), s));
    OSB_CUDA_CHECK(cudaMemsetAsync(w.status, 0, sizeof(uint32_t) * status_words, s));
    const int hblocks = blocks < 1184 ? blocks : 1184;
    k_histogram<K><<<hblocks, 256, 0, s>>>(keys_in, n, passes, w.hist);
    k_scan_hist<<<passes, kBins, 0, s>>>(w.hist, w.base);
    OSB_LAUNCHED(2);
    // Constant digits would be a pure copy; detect them on the host from the histogram.
    std::vector<uint32_t> h(static_cast<size_t>(passes) * kBins);
    OSB_CUDA_CHECK(cudaMemcpyAsync(h.data(), w.hist, h.size() * sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
    OSB_CUDA_CHECK(cudaStreamSynchronize(s));
    bool flipped = false;
    for (int p = 0; p < passes; ++p) {
        bool constant = false;
        for (int d = 0; d < kBins; ++d)
            if (h[static_cast<size_t>(p) * kBins + d] == static_cast<uint32_t>(n)) constant = true;
        if (constant) continue;
        K* ki = flipped ? keys_out : keys_in;
        K* ko = flipped ? keys_in : keys_out;
        uint32_t* vi = flipped ? vals_out : vals_in;
        uint32_t* vo = flipped ? vals_in : vals_out;
        k_onesweep<K><<<blocks, kSortThreads, 0, s>>>(ki, vi, ko, vo, n, p * kRadixBits, w.base + p * kBins,
                                                       w.status + static_cast<size_t>(p) * blocks * kBins,
                                                       w.counter + p);
        OSB_LAUNCHED(1);
        flipped = !flipped;
    }
    return flipped;
}

}  // namespace

size_t radix_workspace_bytes(int n_max, int /*key_bytes*/) {
    const size_t blocks = (static_cast<size_t>(n_max) + kTileKeys - 1) / kTileKeys;
    return sizeof(uint32_t) * (16 * kBins + 64 + 8 * blocks * kBins) + 256;
}

bool radix_sort_u64(uint64_t* ki, uint64_t* ko, uint32_t* vi, uint32_t* vo, int n, int bits, void* ws,
                    cudaStream_t s) {
    return radix_sort<uint64_t>(ki, ko, vi, vo, n, bits, ws, s);
}
bool radix_sort_u32(uint32_t* ki, uint32_t* ko, uint32_t* vi, uint32_t* vo, int n, int bits, void* ws,
                    cudaStream_t s) {
    return radix_sort<uint32_t>(ki, ko, vi, vo, n, bits, ws, s);
}

void launch_iota(uint32_t* v, int n, cudaStream_t s) {
    if (n <= 0) return;
    k_iota<<<(n + 255) / 256, 256, 0, s>>>(v, n);
    OSB_LAUNCHED(1);
}

size_t scan_workspace_bytes(int n) {
    const size_t blocks = (static_cast<size_t>(n) + kScanTile - 1) / kScanTile;
    return sizeof(uint32_t) * (blocks + 64);
}

void launch_gather_scan(const uint32_t* touched, const uint32_t* order, uint32_t* offsets, uint32_t* total, int n,
                        void* ws, cudaStream_t s) {
    if (n <= 0) {
        OSB_CUDA_CHECK(cudaMemsetAsync(total, 0, sizeof(uint32_t), s));
        return;
    }
    const int blocks = (n + kScanTile - 1) / kScanTile;
    uint32_t* counter = static_cast<uint32_t*>(ws);
    uint32_t* status = counter + 64;
    OSB_CUDA_CHECK(cudaMemsetAsync(ws, 0, sizeof(uint32_t) * (blocks + 64), s));
    k_gather_scan<<<blocks, kScanThreads, 0, s>>>(touched, order, offsets, total, n, status, counter);
    OSB_LAUNCHED(1);
}

void launch_emit(const uint32_t* order, const uint32_t* offsets, const uint32_t* touched, const int4* rect, int n,
                 int tiles_x, uint32_t* keys, uint32_t* vals, cudaStream_t s) {
    if (n <= 0) return;
    k_emit<<<(n + 255) / 256, 256, 0, s>>>(order, offsets, touched, rect, n, tiles_x, keys, vals);
    OSB_LAUNCHED(1);
}

void launch_ranges(const uint32_t* sorted_tiles, int m, uint2* ranges, cudaStream_t s) {
    if (m <= 0) return;
    k_ranges<<<(m + 255) / 256, 256, 0, s>>>(sorted_tiles, m, ranges);
    OSB_LAUNCHED(1);
}

}  // namespace osb
