// engine.cu — host orchestration of K1..K5 on one device and one CUDA stream.
//
// Memory layout in HBM: parameters, gradients and Adam moments are four
// planes x stride FP32 buffers (SoA planes, stride = n rounded up to 32 -> every plane starts on
// a 128-B line); per-frame workspaces are pooled and grow monotonically, so steady-state frames
// allocate nothing.
#include <cmath>
#include <cstring>
#include <random>
#include <stdexcept>

#include "engine.h"

namespace osb {

namespace {
long long g_launches = 0;
}

void count_launches(int k) { __atomic_add_fetch(&g_launches, k, __ATOMIC_RELAXED); }
long long launches_total() { return __atomic_load_n(&g_launches, __ATOMIC_RELAXED); }

DevBuf::~DevBuf() {
    if (p_) cudaFree(p_);
}

void DevBuf::ensure(size_t bytes) {
    if (bytes <= cap_ && p_) return;
    const size_t old_cap = p_ ? cap_ : 0;
    if (p_) {
        OSB_CUDA_CHECK(cudaFree(p_));
        p_ = nullptr;
    }
    cap_ = old_cap;
    size_t want = bytes < 256 ? 256 : bytes;
    // a buffer that has to grow grows by at least 25%: a cloud densified every 100 iterations (or
    // a frame whose instance count creeps up) reallocates O(log) times instead of at every step
    // (cudaFree synchronises the device)
    const size_t grown = cap_ + cap_ / 4;
    if (cap_ > 0 && want < grown) want = grown;
    want = (want + 255) & ~size_t(255);
    OSB_CUDA_CHECK(cudaMalloc(&p_, want));
    cap_ = want;
}

DeviceGuard::DeviceGuard(int dev) {
    OSB_CUDA_CHECK(cudaGetDevice(&prev));
    if (prev != dev) OSB_CUDA_CHECK(cudaSetDevice(dev));
}
DeviceGuard::~DeviceGuard() { cudaSetDevice(prev); }

Frame::~Frame() {
    if (ready) cudaEventDestroy(ready);
    if (info_host) cudaFreeHost(info_host);
}

PreprocessOut Frame::pp() const {
    PreprocessOut o;
    o.depth_key = depth_key.as<uint64_t>();
    o.depth_key32 = depth_key32.as<uint32_t>();
    o.depth_range = depth_range.as<uint32_t>();
    o.touched = touched.as<uint32_t>();
    o.rect = rect.as<int4>();
    o.pxy = pxy.as<double2>();
    o.conic_o = conic_o.as<double4>();
    o.splat = splat.as<Splat32>();
    o.radius = radius.as<float>();
    return o;
}

FrameBuffers Frame::fb() const {
    FrameBuffers b;
    b.rgb = rgb.as<float>();
    b.T = T.as<float>();
    b.contrib = contrib.as<int>();
    b.last = last.as<int>();
    b.visited = count_work ? visited.as<int>() : nullptr;
    return b;
}

const char* kernel_name(int id) {
    static const char* names[kKernelCount] = {"preprocess", "depth_sort", "scan_emit", "emit",
                                              "tile_sort",  "ranges",     "blend", "loss",
                                              "bwd_pixels", "bwd_gauss",  "adam"};
    return id >= 0 && id < kKernelCount ? names[id] : "";
}

cudaEvent_t Engine::ev_get() {
    if (!events_.empty()) {
        cudaEvent_t e = events_.back();
        events_.pop_back();
        return e;
    }
    cudaEvent_t e;
    OSB_CUDA_CHECK(cudaEventCreate(&e));
    return e;
}

Engine::Span::Span(Engine& eng, int kind) : e(eng), k(kind) {
    if (!e.timing_) return;
    a = e.ev_get();
    OSB_CUDA_CHECK(cudaEventRecord(a, e.stream_));
}

Engine::Span::~Span() {
    if (!a) return;
    cudaEvent_t b = e.ev_get();
    cudaEventRecord(b, e.stream_);
    e.pending_.push_back({k, a, b});
}

void Engine::collect() {
    for (const Ev& ev : pending_) {
        float ms = 0.0f;
        OSB_CUDA_CHECK(cudaEventSynchronize(ev.b));
        OSB_CUDA_CHECK(cudaEventElapsedTime(&ms, ev.a, ev.b));
        prof_ms_[ev.k] += ms;
        prof_n_[ev.k] += 1;
        events_.push_back(ev.a);
        events_.push_back(ev.b);
    }
    pending_.clear();
}

void Engine::set_profiling(bool timing, bool count_work) {
    DeviceGuard g(device_);
    collect();
    timing_ = timing;
    count_work_ = count_work;
}

void Engine::profile_read(double* ms, long* launches, bool reset) {
    DeviceGuard g(device_);
    collect();
    for (int i = 0; i < kKernelCount; ++i) {
        if (ms) ms[i] = prof_ms_[i];
        if (launches) launches[i] = prof_n_[i];
        if (reset) {
            prof_ms_[i] = 0.0;
            prof_n_[i] = 0;
        }
    }
}

Engine::Engine(int device, cudaStream_t stream) : device_(device), stream_(stream), own_stream_(stream == nullptr) {
    int count = 0;
    OSB_CUDA_CHECK(cudaGetDeviceCount(&count));
    if (device < 0 || device >= count) throw std::invalid_argument("no CUDA device " + std::to_string(device));
    DeviceGuard g(device_);
    if (own_stream_) OSB_CUDA_CHECK(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
}

Engine::~Engine() {
    cudaSetDevice(device_);
    cudaStreamSynchronize(stream_);
    comm_.reset();
    pool_.clear();
    for (const Ev& ev : pending_) {
        cudaEventDestroy(ev.a);
        cudaEventDestroy(ev.b);
    }
    for (cudaEvent_t e : events_) cudaEventDestroy(e);
    if (d2h_stream_) {
        cudaStreamSynchronize(d2h_stream_);
        cudaStreamDestroy(d2h_stream_);
    }
    for (cudaEvent_t e : band_ev_) cudaEventDestroy(e);
    if (copy_stream_) {
        cudaStreamSynchronize(copy_stream_);
        cudaEventDestroy(target_ready_);
        cudaEventDestroy(target_free_);
        cudaStreamDestroy(copy_stream_);
    }
    if (own_stream_) cudaStreamDestroy(stream_);
}

void Engine::upload(const HostCloud& c) {
    DeviceGuard g(device_);
    if (c.sh_degree < 0 || c.sh_degree > 3) throw std::invalid_argument("sh_degree must be in 0..3");
    n_ = c.n();
    ++generation_;
    sh_degree_ = c.sh_degree;
    active_ = c.active_sh_degree < 0 ? 0 : (c.active_sh_degree > c.sh_degree ? c.sh_degree : c.active_sh_degree);
    const int bc = c.bc();
    const Planes pl{bc};
    planes_ = pl.count();
    stride_ = ((n_ > 0 ? n_ : 1) + 31) & ~size_t(31);
    const size_t elems = static_cast<size_t>(planes_) * stride_;
    std::vector<float> host(elems, 0.0f);
    for (size_t i = 0; i < n_; ++i) {
        for (int k = 0; k < 3; ++k) host[k * stride_ + i] = static_cast<float>(c.positions[3 * i + k]);
        for (int b = 0; b < bc; ++b)
            for (int k = 0; k < 3; ++k)
                host[pl.sh(b, k) * stride_ + i] = static_cast<float>(c.sh[(i * bc + b) * 3 + k]);
        for (int k = 0; k < 4; ++k) host[pl.rot(k) * stride_ + i] = static_cast<float>(c.rotations[4 * i + k]);
        for (int k = 0; k < 3; ++k) host[pl.lscale(k) * stride_ + i] = static_cast<float>(c.log_scales[3 * i + k]);
        host[pl.opacity() * stride_ + i] = static_cast<float>(c.opacity[i]);
    }
    params_.ensure(elems * 4);
    grads_.ensure(elems * 4);
    m_.ensure(elems * 4);
    v_.ensure(elems * 4);
    loss_sum_.ensure(64);
    OSB_CUDA_CHECK(cudaMemcpyAsync(params_.as<float>(), host.data(), elems * 4, cudaMemcpyHostToDevice, stream_));
    OSB_CUDA_CHECK(cudaMemsetAsync(grads_.as<float>(), 0, elems * 4, stream_));
    OSB_CUDA_CHECK(cudaMemsetAsync(m_.as<float>(), 0, elems * 4, stream_));
    OSB_CUDA_CHECK(cudaMemsetAsync(v_.as<float>(), 0, elems * 4, stream_));
    reset_per_gaussian_state();
    grads_zero_ = true;
    adam_step_ = 0;
    OSB_CUDA_CHECK(cudaStreamSynchronize(stream_));
}

void Engine::reset_per_gaussian_state() {
    acc_.ensure(stride_ * 48);
    d_screen_.ensure(stride_ * 8);
    norm_sum_.ensure(stride_ * 8);
    hits_.ensure(stride_ * 4);
    max_radius_.ensure(stride_ * 4);
    OSB_CUDA_CHECK(cudaMemsetAsync(d_screen_.as<float>(), 0, stride_ * 8, stream_));
    OSB_CUDA_CHECK(cudaMemsetAsync(norm_sum_.as<double>(), 0, stride_ * 8, stream_));
    OSB_CUDA_CHECK(cudaMemsetAsync(hits_.as<int>(), 0, stride_ * 4, stream_));
    OSB_CUDA_CHECK(cudaMemsetAsync(max_radius_.as<float>(), 0, stride_ * 4, stream_));
}

HostCloud Engine::download() {
    DeviceGuard g(device_);
    HostCloud c;
    c.sh_degree = sh_degree_;
    c.active_sh_degree = active_;
    const int bc = c.bc();
    const Planes pl{bc};
    const size_t elems = static_cast<size_t>(planes_) * stride_;
    std::vector<float> host(elems);
    OSB_CUDA_CHECK(cudaMemcpyAsync(host.data(), params_.as<float>(), elems * 4, cudaMemcpyDeviceToHost, stream_));
    OSB_CUDA_CHECK(cudaStreamSynchronize(stream_));
    c.positions.resize(n_ * 3);
    c.sh.resize(n_ * bc * 3);
    c.rotations.resize(n_ * 4);
    c.log_scales.resize(n_ * 3);
    c.opacity.resize(n_);
    for (size_t i = 0; i < n_; ++i) {
        for (int k = 0; k < 3; ++k) c.positions[3 * i + k] = host[k * stride_ + i];
        for (int b = 0; b < bc; ++b)
            for (int k = 0; k < 3; ++k) c.sh[(i * bc + b) * 3 + k] = host[pl.sh(b, k) * stride_ + i];
        for (int k = 0; k < 4; ++k) c.rotations[4 * i + k] = host[pl.rot(k) * stride_ + i];
        for (int k = 0; k < 3; ++k) c.log_scales[3 * i + k] = host[pl.lscale(k) * stride_ + i];
        c.opacity[i] = host[pl.opacity() * stride_ + i];
    }
    return c;
}

void Engine::set_active_sh_degree(int d) {
    if (d < 0 || d > sh_degree_) throw std::invalid_argument("active_sh_degree out of range");
    active_ = d;
}

static int bits_for(uint64_t v) {
    int b = 0;
    while (b < 64 && (1ull << b) < v) ++b;
    return b;
}

Frame* Engine::render(const double pose12[12], int W, int H, const double bg[3]) {
    DeviceGuard g(device_);
    Frame* f;
    if (!free_.empty()) {
        f = free_.back();
        free_.pop_back();
    } else {
        pool_.emplace_back(new Frame());
        f = pool_.back().get();
    }
    try {
        f->W = W;
        f->H = H;
        f->tiles_x = (W + kTile - 1) / kTile;
        f->tiles_y = (H + kTile - 1) / kTile;
        f->n = static_cast<int>(n_);
        f->generation = generation_;
        f->active_degree = active_;
        std::memcpy(f->pose12, pose12, sizeof(double) * 12);
        for (int i = 0; i < 9; ++i) f->pose.R[i] = pose12[i];
        for (int i = 0; i < 3; ++i) f->pose.t[i] = pose12[9 + i];
        for (int i = 0; i < 3; ++i) f->bg[i] = static_cast<float>(bg ? bg[i] : 0.0);
        f->full_depth_sort = false;
        f->projected = f->given_grid = false;
        render_into(f);
    } catch (...) {
        free_.push_back(f);
        throw;
    }
    return f;
}

Frame* Engine::render_projected(const double* planes, size_t n, int W, int H, const double bg[3],
                                const std::vector<uint2>* ranges, const std::vector<uint32_t>* slots) {
    DeviceGuard g(device_);
    if (n > static_cast<size_t>(INT32_MAX / kSplatPlanes)) throw std::invalid_argument("too many projections");
    Frame* f;
    if (!free_.empty()) {
        f = free_.back();
        free_.pop_back();
    } else {
        pool_.emplace_back(new Frame());
        f = pool_.back().get();
    }
    try {
        f->W = W;
        f->H = H;
        f->tiles_x = (W + kTile - 1) / kTile;
        f->tiles_y = (H + kTile - 1) / kTile;
        f->n = static_cast<int>(n);
        f->generation = generation_;
        f->active_degree = active_;
        for (int i = 0; i < 12; ++i) f->pose12[i] = (i == 0 || i == 4 || i == 8) ? 1.0 : 0.0;
        for (int i = 0; i < 9; ++i) f->pose.R[i] = f->pose12[i];
        for (int i = 0; i < 3; ++i) f->pose.t[i] = 0.0;
        for (int i = 0; i < 3; ++i) f->bg[i] = static_cast<float>(bg ? bg[i] : 0.0);
        f->full_depth_sort = false;
        f->projected = true;
        f->given_grid = ranges != nullptr;
        f->import.ensure(std::max<size_t>(n, 1) * kSplatPlanes * 8);
        if (n)
            OSB_CUDA_CHECK(cudaMemcpyAsync(f->import.as<double>(), planes, n * kSplatPlanes * 8, cudaMemcpyHostToDevice,
                                           stream_));
        if (f->given_grid) {
            f->grid_ranges = *ranges;
            f->grid_slots = *slots;
        } else {
            f->grid_ranges.clear();
            f->grid_slots.clear();
        }
        render_into(f);
    } catch (...) {
        free_.push_back(f);
        throw;
    }
    return f;
}

// The frame's kernels are all enqueued without a host synchronisation: the instance count M is only
// known on the device when the tile sort runs, so the sort, ranges and blend cover min(M, capacity)
// (device-side count, grids sized by the capacity). {M, long-run flag} are copied back
// asynchronously; the first consumer of the frame (validate) checks them and, in the rare case of
// an overflow or a long run of equal FP32 depth keys, grows the buffers / switches to the exact
// 64-bit depth sort and renders the frame again.
#ifndef OSB_HWC_BANDS
#define OSB_HWC_BANDS 8  // render_hwc: bands of tile rows (the D2H of 50 MB of doubles is the bound)
#endif
void Engine::render_into(Frame* f) {
    ++renders_;
    const int W = f->W, H = f->H;
    const size_t n = f->n > 0 ? static_cast<size_t>(f->n) : 1;
    const size_t pixels = static_cast<size_t>(W) * H;
    const int tiles = f->tiles_x * f->tiles_y;
    f->depth_key.ensure(n * 8);
    f->depth_key32.ensure(n * 4);
    f->depth_range.ensure(8);
    f->touched.ensure(n * 4);
    f->rect.ensure(n * 16);
    f->pxy.ensure(n * 16);
    f->conic_o.ensure(n * 32);
    f->splat.ensure(n * sizeof(Splat32));
    f->radius.ensure(n * 4);
    for (int k = 0; k < 2; ++k) {
        f->okeys[k].ensure(n * 8);
        f->ovals[k].ensure(n * 4);
    }
    f->offsets.ensure(n * 4);
    f->total.ensure(16);
    f->ranges.ensure(static_cast<size_t>(tiles) * 8);
    f->rgb.ensure(pixels * 12);
    f->T.ensure(pixels * 4);
    f->contrib.ensure(pixels * 4);
    f->last.ensure(pixels * 4);
    f->count_work = count_work_;
    if (count_work_) {
        f->visited.ensure(pixels * 4);
        f->work.ensure(16);
    }
    f->scan_ws.ensure(scan_workspace_bytes(static_cast<int>(n)));
    if (!f->info_host) OSB_CUDA_CHECK(cudaMallocHost(&f->info_host, 64));
    if (!f->ready) OSB_CUDA_CHECK(cudaEventCreateWithFlags(&f->ready, cudaEventDisableTiming));

    const PreprocessOut pp = f->pp();
    const int N = f->n;
    // one workspace for both sorts, sized for both up front (the zeroed digit totals must survive)
    f->sort_ws.ensure(std::max(radix_workspace_bytes(static_cast<int>(n), 8),
                               radix_workspace_bytes(static_cast<int>(f->ikeys[0].capacity() / 4), 4)));
    uint32_t* long_run_flag = f->total.as<uint32_t>() + 1;
    // K1 clears the frame's K2 scratch on the way (an import of host records or an empty cloud: a
    // separate k_k2_zero below)
    const bool k1_zeroes = !f->projected && N > 0 && !f->given_grid;
    // K1 (or the import of host projection records)
    {
        Span sp(*this, kPreprocess);
        OSB_CUDA_CHECK(cudaMemsetAsync(pp.depth_range, 0xFF, 8, stream_));
        if (f->projected)
            launch_import_projections(f->import.as<double>(), N, W, H, pp, stream_);
        else
            launch_preprocess(params_.as<float>(), N, static_cast<int>(stride_), (sh_degree_ + 1) * (sh_degree_ + 1),
                              active_, f->pose, W, H, pp, stream_,
                              k1_zeroes ? k2_scratch(f->sort_ws.as<void>(), long_run_flag, f->ranges.as<uint2>(), tiles,
                                                     f->scan_ws.as<void>(), N)
                                        : K2Scratch{});
    }
    if (f->given_grid) {  // caller-supplied tile lists: no K2
        const uint32_t M = static_cast<uint32_t>(f->grid_slots.size());
        f->ivals[0].ensure(std::max<size_t>(M, 1) * 4);
        if (M)
            OSB_CUDA_CHECK(cudaMemcpyAsync(f->ivals[0].as<uint32_t>(), f->grid_slots.data(), size_t(M) * 4,
                                           cudaMemcpyHostToDevice, stream_));
        OSB_CUDA_CHECK(cudaMemcpyAsync(f->ranges.as<uint2>(), f->grid_ranges.data(), size_t(tiles) * 8,
                                       cudaMemcpyHostToDevice, stream_));
        f->inst_in_alt = false;
        {
            Span sp(*this, kBlend);
            launch_blend(f->inst_gid(), f->ranges.as<uint2>(), pp, W, H, f->tiles_x, f->tiles_y, f->bg, f->fb(),
                         stream_, strict_guard_);
        }
        // the host vectors are read by the copies above: finish them before the caller may free
        OSB_CUDA_CHECK(cudaStreamSynchronize(stream_));
        f->cap = f->M = M;
        f->validated = true;
        return;
    }
    // K2a: depth rank = (t_r, id) order. Fast path: stable sort of the FP32-rounded t_r (monotone)
    // + exact FP64 re-ordering inside runs of equal keys; a run longer than 64 raises a flag
    // and validate() renders the frame again with the full 64-bit sort.
    const uint32_t* order;
    const uint32_t* keys24 = nullptr;  // fast path: the sorted 24-bit keys (runs fixed in the emission)
    {
        Span sp(*this, kDepthSort);
        if (!k1_zeroes)
            launch_k2_zero(f->sort_ws.as<void>(), long_run_flag, f->ranges.as<uint2>(), tiles, f->scan_ws.as<void>(),
                           static_cast<int>(N), stream_);
        bool flipped;
        if (f->full_depth_sort) {
            flipped = radix_sort_u64(f->okeys[0].as<uint64_t>(), f->okeys[1].as<uint64_t>(), f->ovals[0].as<uint32_t>(),
                                     f->ovals[1].as<uint32_t>(), N, 64, f->sort_ws.as<void>(), stream_, pp.depth_key,
                                     true, true);
        } else {
            uint32_t* k32[2] = {f->okeys[0].as<uint32_t>(), f->okeys[1].as<uint32_t>()};
            flipped = radix_sort_depth24(pp.depth_key32, pp.depth_range, k32[0], k32[1], f->ovals[0].as<uint32_t>(),
                                         f->ovals[1].as<uint32_t>(), N, f->sort_ws.as<void>(), stream_, true);
            keys24 = k32[flipped ? 1 : 0];
        }
        order = f->ovals[flipped ? 1 : 0].as<uint32_t>();
    }
    // K2b: scan of tiles_touched in depth order + balanced (tile, gid) emission. A frame with no
    // instance buffer yet sizes it first (one synchronous counting pass).
    if (f->ikeys[0].capacity() == 0) {
        launch_scan_emit(pp.touched, order, pp.rect, N, f->tiles_x, nullptr, nullptr, 0, f->total.as<uint32_t>(),
                         f->scan_ws.as<void>(), nullptr, nullptr, stream_, keys24, pp.depth_key, long_run_flag);
        uint32_t host = 0;
        OSB_CUDA_CHECK(cudaMemcpyAsync(&host, f->total.as<uint32_t>(), 4, cudaMemcpyDeviceToHost, stream_));
        scan_sums_reset(f->scan_ws.as<void>(), static_cast<int>(N), stream_);  // the emission below adds again
        OSB_CUDA_CHECK(cudaStreamSynchronize(stream_));
        grow_instances(f, host);
    }
    const uint32_t cap = static_cast<uint32_t>(f->ikeys[0].capacity() / 4);
    f->cap = cap;
    f->emit_first.ensure((static_cast<size_t>(emit_ctas(cap)) + 1) * 4);
    // the emission also does the tile sort's first upsweep (tiles <= 2^16: two 8-bit passes)
    const int tile_bits = bits_for(static_cast<uint64_t>(tiles));
    const bool fused_counts = tile_bits <= 16;
    const void* ws_zeroed = f->sort_ws.as<void>();
    f->sort_ws.ensure(radix_workspace_bytes(static_cast<int>(cap), 4));
    {
        Span sp(*this, kScan);
        // the first frame's instance buffer can grow the workspace: its tile slot is zeroed again
        if (f->sort_ws.as<void>() != ws_zeroed) tile_sort_prepare(f->sort_ws.as<void>(), stream_);
        launch_scan_emit(pp.touched, order, pp.rect, N, f->tiles_x, f->ikeys[0].as<uint32_t>(),
                         f->ivals[0].as<uint32_t>(), cap, f->total.as<uint32_t>(), f->scan_ws.as<void>(),
                         f->emit_first.as<uint32_t>(), fused_counts ? f->sort_ws.as<void>() : nullptr, stream_, keys24,
                         pp.depth_key, long_run_flag);
    }
    // {M, long-run flag} are final here: read them back now so validate() only waits for this
    // point of the frame, not for the blend
    OSB_CUDA_CHECK(cudaMemcpyAsync(f->info_host, f->total.as<uint32_t>(), 8, cudaMemcpyDeviceToHost, stream_));
    OSB_CUDA_CHECK(cudaEventRecord(f->ready, stream_));
    // K2c: stable sort by tile over min(M, cap) instances (count read on the device); its last pass
    // writes the tile ranges instead of the sorted keys
    {
        Span sp(*this, kTileSort);
        f->inst_in_alt = radix_sort_u32(f->ikeys[0].as<uint32_t>(), f->ikeys[1].as<uint32_t>(),
                                        f->ivals[0].as<uint32_t>(), f->ivals[1].as<uint32_t>(), static_cast<int>(cap),
                                        tile_bits, f->sort_ws.as<void>(), stream_, f->total.as<uint32_t>(),
                                        fused_counts, true, f->ranges.as<uint2>());  // + the tile ranges
    }
    // K3 (render_hwc: in bands of tile rows, each band's host copy queued behind it on the D2H stream)
    {
        Span sp(*this, kBlend);
        if (!hwc_host_) {
            launch_blend(f->inst_gid(), f->ranges.as<uint2>(), pp, W, H, f->tiles_x, f->tiles_y, f->bg, f->fb(),
                         stream_, strict_guard_);
        } else {
            constexpr int kBands = OSB_HWC_BANDS;
            const size_t plane = pixels;
            hwc_.ensure(plane * 3 * sizeof(double));
            if (!d2h_stream_) OSB_CUDA_CHECK(cudaStreamCreateWithFlags(&d2h_stream_, cudaStreamNonBlocking));
            while (band_ev_.size() < static_cast<size_t>(kBands)) {
                cudaEvent_t e;
                OSB_CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
                band_ev_.push_back(e);
            }
            for (int b = 0; b < kBands; ++b) {
                const int r0 = f->tiles_y * b / kBands, r1 = f->tiles_y * (b + 1) / kBands;
                if (r1 <= r0) continue;
                launch_blend(f->inst_gid(), f->ranges.as<uint2>(), pp, W, H, f->tiles_x, f->tiles_y, f->bg, f->fb(),
                             stream_, strict_guard_, r0, r1);
                OSB_CUDA_CHECK(cudaEventRecord(band_ev_[b], stream_));
                OSB_CUDA_CHECK(cudaStreamWaitEvent(d2h_stream_, band_ev_[b], 0));
                const size_t p0 = static_cast<size_t>(r0) * kTile * W;
                const size_t p1 = std::min(static_cast<size_t>(r1) * kTile, static_cast<size_t>(H)) * W;
                launch_planar_to_hwc_f64(f->rgb.as<float>(), plane, hwc_.as<double>(), d2h_stream_, p0, p1);
                OSB_CUDA_CHECK(cudaMemcpyAsync(hwc_host_ + 3 * p0, hwc_.as<double>() + 3 * p0,
                                               (p1 - p0) * 3 * sizeof(double), cudaMemcpyDeviceToHost, d2h_stream_));
            }
        }
    }
    f->validated = false;
    f->M = cap;  // provisional until validate()
}

void Engine::grow_instances(Frame* f, uint32_t M) {
    const size_t want = (static_cast<size_t>(M) + M / 4 + 1024) * 4;
    if (want <= f->ikeys[0].capacity()) return;
    OSB_CUDA_CHECK(cudaStreamSynchronize(stream_));  // the buffers may still be in use
    for (int k = 0; k < 2; ++k) {
        f->ikeys[k].ensure(want);
        f->ivals[k].ensure(want);
    }
}

void Engine::validate(Frame* f) {
    if (!f || f->validated) return;
    DeviceGuard g(device_);
    for (int attempt = 0; attempt < 3; ++attempt) {
        OSB_CUDA_CHECK(cudaEventSynchronize(f->ready));
        const uint32_t M = f->n == 0 ? 0u : f->info_host[0];
        const bool long_run = f->info_host[1] != 0 && !f->full_depth_sort;
        if (M <= f->cap && !long_run) {
            f->M = M;
            f->validated = true;
            return;
        }
        if (long_run) f->full_depth_sort = true;
        grow_instances(f, M);
        render_into(f);
    }
    throw std::runtime_error("render: instance buffer sizing did not converge");
}

void Engine::projection_detail(Frame* f, std::vector<double>& out) {
    DeviceGuard g(device_);
    validate(f);
    if (f->projected || static_cast<size_t>(f->n) != n_ || f->generation != generation_)
        throw std::logic_error("StateMismatch: render output does not match the cloud");
    const size_t n = static_cast<size_t>(f->n);
    out.assign(n * 6, 0.0);
    if (!n) return;
    DevBuf tmp;
    tmp.ensure(n * 6 * 8);
    launch_projection_detail(params_.as<float>(), f->n, static_cast<int>(stride_), (sh_degree_ + 1) * (sh_degree_ + 1),
                             f->pose, f->W, f->H, tmp.as<double>(), stream_);
    OSB_CUDA_CHECK(cudaMemcpyAsync(out.data(), tmp.as<double>(), n * 6 * 8, cudaMemcpyDeviceToHost, stream_));
    OSB_CUDA_CHECK(cudaStreamSynchronize(stream_));
}

void Engine::release(Frame* f) {
    if (!f) return;
    // a frame released unread still tells the pool how large the instance buffers must be
    if (!f->validated) {
        DeviceGuard g(device_);
        OSB_CUDA_CHECK(cudaEventSynchronize(f->ready));
        if (f->n > 0 && f->info_host[0] > f->cap) grow_instances(f, f->info_host[0]);
        f->validated = true;
    }
    free_.push_back(f);
}

void Engine::backward(Frame* f, const float* d_image, bool accumulate) {
    DeviceGuard g(device_);
    validate(f);
    if (f->projected || static_cast<size_t>(f->n) != n_ || f->generation != generation_)
        throw std::logic_error("StateMismatch: render output does not match the cloud");
    // K4b overwrites (no read of the gradient planes, zeros for culled Gaussians) when the buffer is
    // logically zero or the caller asks for reference overwrite semantics.
    const bool overwrite = !accumulate || grads_zero_;
    OSB_CUDA_CHECK(cudaMemsetAsync(acc_.as<float4>(), 0, stride_ * 48, stream_));
    const PreprocessOut pp = f->pp();
    {
        Span sp(*this, kBwdPixels);
        if (deterministic_) {
            det_inst_.ensure(static_cast<size_t>(f->M) * 9 * sizeof(float) + 64);
            det_rank_.ensure(static_cast<size_t>(f->n) * sizeof(uint32_t) + 64);
            OSB_CUDA_CHECK(cudaMemsetAsync(det_inst_.as<float>(), 0, static_cast<size_t>(f->M) * 9 * sizeof(float),
                                           stream_));
            launch_backward_pixels_det(f->inst_gid(), f->ranges.as<uint2>(), pp, f->W, f->H, f->tiles_x, f->tiles_y,
                                       f->bg, f->fb(), d_image, scan_emit_arrays(f->scan_ws.as<void>(), f->n), f->n,
                                       det_rank_.as<uint32_t>(), det_inst_.as<float>(), acc_.as<float4>(), stream_);
        } else {
            launch_backward_pixels(f->inst_gid(), f->ranges.as<uint2>(), pp, f->W, f->H, f->tiles_x, f->tiles_y,
                                   f->bg, f->fb(), d_image, acc_.as<float4>(), stream_);
        }
    }
    ScreenStats st{d_screen_.as<float2>(), norm_sum_.as<double>(), hits_.as<int>()};
    if (!accumulate) OSB_CUDA_CHECK(cudaMemsetAsync(d_screen_.as<float2>(), 0, stride_ * 8, stream_));
    {
        Span sp(*this, kBwdGauss);
        launch_backward_gaussians(params_.as<float>(), f->n, static_cast<int>(stride_),
                                  (sh_degree_ + 1) * (sh_degree_ + 1), f->active_degree, f->pose, f->W, f->H,
                                  pp, acc_.as<float4>(), grads_.as<float>(), st, overwrite, stream_);
    }
    grads_zero_ = false;
}

void Engine::materialize_grads() {
    if (!grads_zero_) return;
    OSB_CUDA_CHECK(cudaMemsetAsync(grads_.as<float>(), 0, static_cast<size_t>(planes_) * stride_ * 4, stream_));
    // the planes now hold real zeros: a caller may write them directly (collectives, uploads) and
    // the next consumer must not clear them again
    grads_zero_ = false;
}

float* Engine::d_image_buffer(size_t pixels) {
    d_image_.ensure(pixels * 12);
    return d_image_.as<float>();
}

float* Engine::gt_buffer(size_t pixels) {
    gt_.ensure(pixels * 12);
    return gt_.as<float>();
}

const float* Engine::upload_target_async(const float* host, size_t pixels) {
    DeviceGuard g(device_);
    if (!copy_stream_) {
        OSB_CUDA_CHECK(cudaStreamCreateWithFlags(&copy_stream_, cudaStreamNonBlocking));
        OSB_CUDA_CHECK(cudaEventCreateWithFlags(&target_ready_, cudaEventDisableTiming));
        OSB_CUDA_CHECK(cudaEventCreateWithFlags(&target_free_, cudaEventDisableTiming));
        OSB_CUDA_CHECK(cudaEventRecord(target_free_, stream_));
    }
    if (gt_.capacity() < pixels * 12) {
        OSB_CUDA_CHECK(cudaStreamSynchronize(copy_stream_));
        OSB_CUDA_CHECK(cudaStreamSynchronize(stream_));
    }
    float* buf = gt_buffer(pixels);
    OSB_CUDA_CHECK(cudaStreamWaitEvent(copy_stream_, target_free_, 0));  // previous consumer done
    OSB_CUDA_CHECK(cudaMemcpyAsync(buf, host, pixels * 12, cudaMemcpyHostToDevice, copy_stream_));
    OSB_CUDA_CHECK(cudaEventRecord(target_ready_, copy_stream_));
    return buf;
}

void Engine::wait_target() { OSB_CUDA_CHECK(cudaStreamWaitEvent(stream_, target_ready_, 0)); }

void Engine::release_target() { OSB_CUDA_CHECK(cudaEventRecord(target_free_, stream_)); }

double Engine::loss(Frame* f, const float* gt, double lambda, double mask_bottom_fraction, bool want_value) {
    DeviceGuard g(device_);
    validate(f);
    const size_t pixels = static_cast<size_t>(f->W) * f->H;
    float* dimg = d_image_buffer(pixels);
    const int masked = static_cast<int>(std::floor(mask_bottom_fraction * f->H));
    const int keep = f->H - masked;
    if (lambda > 0.0) ssim_planes_.ensure(pixels * 9 * sizeof(float));
    {
        Span sp(*this, kLoss);
        launch_loss(f->fb().rgb, gt, f->W, f->H, keep, lambda, dimg, ssim_planes_.as<float>(), loss_sum_.as<double>(),
                    stream_);
    }
    last_lambda_ = lambda;
    if (!want_value) return 0.0;
    return loss_value(f, mask_bottom_fraction);
}

double Engine::loss_value(const Frame* f, double mask_bottom_fraction) {
    DeviceGuard g(device_);
    const int masked = static_cast<int>(std::floor(mask_bottom_fraction * f->H));
    const double npx = static_cast<double>(f->W) * (f->H - masked);
    const double n = npx * 3.0;
    double s[4] = {0, 0, 0, 0};
    OSB_CUDA_CHECK(cudaMemcpyAsync(s, loss_sum_.as<double>(), 32, cudaMemcpyDeviceToHost, stream_));
    OSB_CUDA_CHECK(cudaStreamSynchronize(stream_));
    // trainer.cpp:54-63: (1 - l) * L1 + l * (1 - SSIM), SSIM = mean over channels of the pixel mean
    double value = (1.0 - last_lambda_) * (s[0] / n);
    if (last_lambda_ > 0.0) value += last_lambda_ * (1.0 - ((s[1] + s[2] + s[3]) / npx) / 3.0);
    return value;
}

const double* Engine::image_hwc_device(Frame* f) {
    DeviceGuard g(device_);
    validate(f);
    const size_t plane = static_cast<size_t>(f->W) * f->H;
    hwc_.ensure(plane * 3 * sizeof(double));
    launch_planar_to_hwc_f64(f->rgb.as<float>(), plane, hwc_.as<double>(), stream_);
    return hwc_.as<double>();
}

Frame* Engine::render_hwc(const double pose12[12], int W, int H, const double bg[3], double* host) {
    DeviceGuard g(device_);
    hwc_host_ = host;
    Frame* f = nullptr;
    try {
        f = render(pose12, W, H, bg);
    } catch (...) {
        hwc_host_ = nullptr;
        if (d2h_stream_) cudaStreamSynchronize(d2h_stream_);
        throw;
    }
    hwc_host_ = nullptr;
    try {
        const unsigned long before = renders_;
        validate(f);  // a re-render (instance overflow, long depth run) blends in one launch, no copies
        OSB_CUDA_CHECK(cudaStreamSynchronize(d2h_stream_));
        if (renders_ != before) image_hwc(f, host);  // the banded copies held the first attempt
    } catch (...) {
        if (d2h_stream_) cudaStreamSynchronize(d2h_stream_);
        release(f);
        throw;
    }
    return f;
}

void Engine::image_hwc(Frame* f, double* host) {
    DeviceGuard g(device_);
    validate(f);
    const size_t plane = static_cast<size_t>(f->W) * f->H;
    hwc_.ensure(plane * 3 * sizeof(double));
    launch_planar_to_hwc_f64(f->rgb.as<float>(), plane, hwc_.as<double>(), stream_);
    OSB_CUDA_CHECK(cudaMemcpyAsync(host, hwc_.as<double>(), plane * 3 * sizeof(double), cudaMemcpyDeviceToHost,
                                   stream_));
    OSB_CUDA_CHECK(cudaStreamSynchronize(stream_));
}

void Engine::loss_sums_async(double* host) {
    DeviceGuard g(device_);
    OSB_CUDA_CHECK(cudaMemcpyAsync(host, loss_sum_.as<double>(), 32, cudaMemcpyDeviceToHost, stream_));
}

void Engine::adam_step(const TrainHyper& h, double extent, long iteration, bool zero_grad, size_t begin,
                       size_t count) {
    DeviceGuard g(device_);
    adam_step_ += 1;
    const double bias1 = 1.0 - std::pow(0.9, static_cast<double>(adam_step_));
    const double bias2 = 1.0 - std::pow(0.999, static_cast<double>(adam_step_));
    double t = 1.0;
    if (h.iterations > 0) {
        t = static_cast<double>(iteration) / h.iterations;
        t = t < 0.0 ? 0.0 : (t > 1.0 ? 1.0 : t);
    }
    const double lr_pos = std::exp((1.0 - t) * std::log(h.lr_position_init * extent) +
                                   t * std::log(h.lr_position_final * extent));
    AdamArgs a;
    const int bc = (sh_degree_ + 1) * (sh_degree_ + 1);
    const Planes pl{bc};
    for (int i = 0; i < 64; ++i) a.lr_plane[i] = 0.0f;
    for (int k = 0; k < 3; ++k) a.lr_plane[k] = static_cast<float>(lr_pos);
    for (int b = 0; b < bc; ++b)
        for (int k = 0; k < 3; ++k) a.lr_plane[pl.sh(b, k)] = static_cast<float>(b == 0 ? h.lr_sh_dc : h.lr_sh_rest);
    for (int k = 0; k < 4; ++k) a.lr_plane[pl.rot(k)] = static_cast<float>(h.lr_rotation);
    for (int k = 0; k < 3; ++k) a.lr_plane[pl.lscale(k)] = static_cast<float>(h.lr_scale);
    a.lr_plane[pl.opacity()] = static_cast<float>(h.lr_opacity);
    a.inv_bias1 = static_cast<float>(1.0 / bias1);
    a.inv_bias2 = static_cast<float>(1.0 / bias2);
    a.planes = planes_;
    a.stride = static_cast<int>(stride_);
    const size_t total = static_cast<size_t>(planes_) * stride_;
    if (begin > total || (begin & 3) != 0) throw std::invalid_argument("adam_step: range start out of bounds");
    if (count > total - begin) count = total - begin;
    if ((count & 3) != 0) throw std::invalid_argument("adam_step: range length must be a multiple of 4");
    a.begin = static_cast<long>(begin);
    a.count = static_cast<long>(count);
    // Consumed gradients are not cleared in memory: the flag makes the next backward overwrite them.
    a.zero_grad = 0;
    materialize_grads();
    {
        Span sp(*this, kAdam);
        launch_adam(params_.as<float>(), grads_.as<float>(), m_.as<float>(), v_.as<float>(), a, stream_);
    }
    if (zero_grad) grads_zero_ = true;
}

void Engine::zero_grad() { grads_zero_ = true; }

void Engine::begin_training(bool fresh) {
    DeviceGuard g(device_);
    reset_per_gaussian_state();
    grads_zero_ = true;
    if (fresh) {
        const size_t bytes = static_cast<size_t>(planes_) * stride_ * 4;
        OSB_CUDA_CHECK(cudaMemsetAsync(m_.as<float>(), 0, bytes, stream_));
        OSB_CUDA_CHECK(cudaMemsetAsync(v_.as<float>(), 0, bytes, stream_));
        adam_step_ = 0;
    }
}

void Engine::reset_screen_stats() {
    DeviceGuard g(device_);
    OSB_CUDA_CHECK(cudaMemsetAsync(norm_sum_.as<double>(), 0, stride_ * 8, stream_));
    OSB_CUDA_CHECK(cudaMemsetAsync(hits_.as<int>(), 0, stride_ * 4, stream_));
}

void Engine::observe(Frame* f) {
    DeviceGuard g(device_);
    validate(f);
    if (f->projected || static_cast<size_t>(f->n) != n_ || f->generation != generation_)
        throw std::logic_error("StateMismatch: render output does not match the cloud");
    launch_observe(f->radius.as<float>(), max_radius_.as<float>(), f->n, stream_);
}

void Engine::reset_opacity(double ceiling) {
    DeviceGuard g(device_);
    const Planes pl{(sh_degree_ + 1) * (sh_degree_ + 1)};
    const double cap = std::log(ceiling / (1.0 - ceiling));  // logit (scene.hpp:58)
    launch_reset_opacity(params_.as<float>() + static_cast<size_t>(pl.opacity()) * stride_, static_cast<int>(n_), cap,
                         stream_);
}

EditSummary Engine::densify_and_prune(const DensifyArgs& a, unsigned long long rng_seed) {
    DeviceGuard g(device_);
    // data-parallel ranks: this rank's statistics are partial sums of its own views, its moments
    // are current only on its shard — make both global first (comm.cpp)
    dp_reduce_stats();
    dp_gather_moments();
    EditSummary e;
    const int n = static_cast<int>(n_);
    const int bc = (sh_degree_ + 1) * (sh_degree_ + 1);
    DevBuf &code = dz_code_, &rank = dz_rank_, &ws = dz_ws_, &csrc = dz_csrc_, &ssrc = dz_ssrc_,
           &normals = dz_normals_, &keep = dz_keep_, &dest = dz_dest_;  // persistent scratch (no per-call malloc/free)
    int nc = 0, ns = 0;
    if (n > 0) {
        code.ensure(static_cast<size_t>(n) * 8);
        rank.ensure(static_cast<size_t>(n) * 8);
        ws.ensure(densify_scan_workspace_bytes(n));
        launch_densify_mark(params_.as<float>(), n, static_cast<int>(stride_), bc, norm_sum_.as<double>(),
                            hits_.as<int>(), a, code.as<unsigned long long>(), stream_);
        launch_exclusive_scan_u64(code.as<unsigned long long>(), rank.as<unsigned long long>(), n, ws.as<void>(),
                                  stream_);
        const size_t nb = (static_cast<size_t>(n) + 1023) / 1024;
        unsigned long long tot = 0;
        OSB_CUDA_CHECK(cudaMemcpyAsync(&tot, ws.as<unsigned long long>() + nb, 8, cudaMemcpyDeviceToHost, stream_));
        OSB_CUDA_CHECK(cudaStreamSynchronize(stream_));
        nc = static_cast<int>(tot & 0xffffffffull);
        ns = static_cast<int>(tot >> 32);
        csrc.ensure(static_cast<size_t>(nc) * 4);
        ssrc.ensure(static_cast<size_t>(ns) * 4);
        launch_densify_sources(code.as<unsigned long long>(), rank.as<unsigned long long>(), n, csrc.as<int>(),
                               ssrc.as<int>(), stream_);
    }
    // The split children's offsets: the reference's own RNG stream (trainer.cpp:215, 227), drawn in
    // its order (split parents ascending, child 0 then 1, x y z) -> bit-identical normals.
    std::vector<double> xi(static_cast<size_t>(ns) * 6);
    {
        std::mt19937_64 rng(rng_seed);
        std::normal_distribution<double> normal(0.0, 1.0);
        for (double& x : xi) x = normal(rng);
    }
    normals.ensure(xi.size() * 8);
    if (!xi.empty())
        OSB_CUDA_CHECK(cudaMemcpyAsync(normals.as<double>(), xi.data(), xi.size() * 8, cudaMemcpyHostToDevice, stream_));
    const long total = static_cast<long>(n) + nc + 2L * ns;
    long kept = 0;
    if (total > 0) {
        keep.ensure(static_cast<size_t>(total) * 8);
        dest.ensure(static_cast<size_t>(total) * 8);
        ws.ensure(densify_scan_workspace_bytes(total));
        launch_densify_keep(params_.as<float>(), n, static_cast<int>(stride_), bc, nc, total,
                            code.as<unsigned long long>(), csrc.as<int>(), ssrc.as<int>(), max_radius_.as<float>(), a,
                            keep.as<unsigned long long>(), stream_);
        launch_exclusive_scan_u64(keep.as<unsigned long long>(), dest.as<unsigned long long>(), total, ws.as<void>(),
                                  stream_);
        const size_t nb = (static_cast<size_t>(total) + 1023) / 1024;
        unsigned long long k = 0;
        OSB_CUDA_CHECK(cudaMemcpyAsync(&k, ws.as<unsigned long long>() + nb, 8, cudaMemcpyDeviceToHost, stream_));
        OSB_CUDA_CHECK(cudaStreamSynchronize(stream_));  // also keeps xi alive until the copy is done
        kept = static_cast<long>(k);
    }
    e.cloned = nc;
    e.split = ns;
    e.pruned = (total - kept) - ns;  // split parents are not "pruned" (trainer.cpp:262)
    e.final_count = static_cast<size_t>(kept);
    // gather into new planes (new stride), then swap them in
    const size_t stride2 = ((kept > 0 ? static_cast<size_t>(kept) : 1) + 31) & ~size_t(31);
    const size_t elems2 = static_cast<size_t>(planes_) * stride2;
    DevBuf &P2 = spare_p_, &M2 = spare_m_, &V2 = spare_v_;  // double-buffered planes: the old ones become the spares
    P2.ensure(elems2 * 4);
    M2.ensure(elems2 * 4);
    V2.ensure(elems2 * 4);
    OSB_CUDA_CHECK(cudaMemsetAsync(P2.as<float>(), 0, elems2 * 4, stream_));
    OSB_CUDA_CHECK(cudaMemsetAsync(M2.as<float>(), 0, elems2 * 4, stream_));
    OSB_CUDA_CHECK(cudaMemsetAsync(V2.as<float>(), 0, elems2 * 4, stream_));
    launch_densify_write(params_.as<float>(), m_.as<float>(), v_.as<float>(), n, static_cast<int>(stride_), bc, nc, total,
                         keep.as<unsigned long long>(), dest.as<unsigned long long>(), csrc.as<int>(), ssrc.as<int>(),
                         normals.as<double>(), a, P2.as<float>(), M2.as<float>(), V2.as<float>(),
                         static_cast<int>(stride2), stream_);
    OSB_CUDA_CHECK(cudaStreamSynchronize(stream_));
    params_.swap(P2);
    m_.swap(M2);
    v_.swap(V2);
    n_ = static_cast<size_t>(kept);
    stride_ = stride2;
    ++generation_;
    // GradientBuffer::resize + DensifyStats::resize (trainer.cpp:268-269): gradients and statistics restart
    grads_.ensure(elems2 * 4);
    grads_zero_ = true;
    reset_per_gaussian_state();
    return e;
}

double Engine::psnr(Frame* f, const float* gt) {
    DeviceGuard g(device_);
    validate(f);
    const long n = 3L * f->W * f->H;
    scratch_.ensure(64);
    launch_sq_err(f->rgb.as<float>(), gt, n, scratch_.as<double>(), stream_);
    double sum = 0.0;
    OSB_CUDA_CHECK(cudaMemcpyAsync(&sum, scratch_.as<double>(), 8, cudaMemcpyDeviceToHost, stream_));
    OSB_CUDA_CHECK(cudaStreamSynchronize(stream_));
    const double cap = 99.0;  // kPsnrCap (metrics.hpp)
    const double mse = sum / static_cast<double>(n);
    if (mse <= 0.0) return cap;
    const double v = 10.0 * std::log10(1.0 / mse);
    return v < cap ? v : cap;
}

void Engine::read_adam(std::vector<float>& m, std::vector<float>& v) {
    DeviceGuard g(device_);
    dp_gather_moments();  // a sharded optimizer's moments are current only on each rank's shard
    const size_t elems = static_cast<size_t>(planes_) * stride_;
    m.resize(elems);
    v.resize(elems);
    OSB_CUDA_CHECK(cudaMemcpyAsync(m.data(), m_.as<float>(), elems * 4, cudaMemcpyDeviceToHost, stream_));
    OSB_CUDA_CHECK(cudaMemcpyAsync(v.data(), v_.as<float>(), elems * 4, cudaMemcpyDeviceToHost, stream_));
    OSB_CUDA_CHECK(cudaStreamSynchronize(stream_));
}

void Engine::write_adam(const std::vector<float>& m, const std::vector<float>& v, long step) {
    DeviceGuard g(device_);
    const size_t elems = static_cast<size_t>(planes_) * stride_;
    if (m.size() != elems || v.size() != elems) throw std::invalid_argument("write_adam: size mismatch");
    OSB_CUDA_CHECK(cudaMemcpyAsync(m_.as<float>(), m.data(), elems * 4, cudaMemcpyHostToDevice, stream_));
    OSB_CUDA_CHECK(cudaMemcpyAsync(v_.as<float>(), v.data(), elems * 4, cudaMemcpyHostToDevice, stream_));
    OSB_CUDA_CHECK(cudaStreamSynchronize(stream_));
    adam_step_ = step;
}

void Engine::synchronize() {
    DeviceGuard g(device_);
    OSB_CUDA_CHECK(cudaStreamSynchronize(stream_));
}

}  // namespace osb
