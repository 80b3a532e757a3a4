// engine.h — device context (parameters, gradients, Adam state) and frame workspaces.
#pragma once

#include <cuda_runtime.h>

#include <memory>
#include <utility>
#include <vector>

#include "kernels.h"

namespace osb {

// Host mirror of the reference GaussianCloud (proj/include/omnisplat/scene.hpp:31-55).
struct HostCloud {
    int sh_degree = 3;
    int active_sh_degree = 0;
    std::vector<double> positions, sh, rotations, log_scales, opacity;
    size_t n() const { return positions.size() / 3; }
    int bc() const { return (sh_degree + 1) * (sh_degree + 1); }
};

// Growable device allocation (never shrinks; reused across frames).
class DevBuf {
public:
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf();
    void ensure(size_t bytes);
    template <typename T>
    T* as() const { return static_cast<T*>(p_); }
    size_t capacity() const { return cap_; }
    void swap(DevBuf& o) {
        std::swap(p_, o.p_);
        std::swap(cap_, o.cap_);
    }

private:
    void* p_ = nullptr;
    size_t cap_ = 0;
};

// Hyper-parameters adam_step reads (trainer.hpp:19-51 TrainConfig subset) + loss settings.
struct TrainHyper {
    long iterations = 7000;
    double lr_position_init = 1.6e-4, lr_position_final = 1.6e-6;
    double lr_sh_dc = 2.5e-3, lr_sh_rest = 2.5e-3 / 20.0;
    double lr_opacity = 5e-2, lr_scale = 5e-3, lr_rotation = 1e-3;
};

// Kernel families timed by the optional CUDA-event profiler (osplat_gpu_profile).
enum KernelId { kPreprocess, kDepthSort, kScan, kEmit, kTileSort, kRanges, kBlend, kLoss, kBwdPixels, kBwdGauss,
                kAdam, kKernelCount };
const char* kernel_name(int id);

// EditSummary (trainer.hpp:93-98).
struct EditSummary {
    long cloned = 0, split = 0, pruned = 0;
    size_t final_count = 0;
};

struct Frame {
    int W = 0, H = 0, tiles_x = 0, tiles_y = 0, n = 0, active_degree = 0;
    unsigned long generation = 0;  // Engine::generation() at render time (parameters' identity)
    uint32_t M = 0;
    double pose12[12];
    Pose pose;
    float bg[3] = {0, 0, 0};
    bool inst_in_alt = false;  // sorted instance gids live in inst_vals[1]
    // per Gaussian (K1 outputs)
    DevBuf depth_key, depth_key32, depth_range, touched, rect, pxy, conic_o, splat, radius;
    bool full_depth_sort = false;  // set when the FP32-key fast path met a long run of equal keys
    uint32_t cap = 0;              // instance capacity the frame was rendered with
    bool validated = true;         // {M, long-run flag} checked (Engine::validate)
    uint32_t* info_host = nullptr; // pinned {M, long-run flag}
    cudaEvent_t ready = nullptr;   // recorded after the frame's kernels and the info read-back
    ~Frame();
    // depth sort
    DevBuf okeys[2], ovals[2], offsets, total;
    // instances
    DevBuf ikeys[2], ivals[2], ranges;
    // pixels
    DevBuf rgb, T, contrib, last, visited, work;
    bool count_work = false;
    DevBuf sort_ws, scan_ws, emit_first;
    // Frames of host-supplied projections (render_projected): no Gaussian parameters behind them,
    // so no backward; `grid_*` hold a caller-supplied tile grid (K2 skipped) when given_grid.
    bool projected = false, given_grid = false;
    DevBuf import;
    std::vector<uint2> grid_ranges;
    std::vector<uint32_t> grid_slots;
    const uint32_t* inst_gid() const { return ivals[inst_in_alt ? 1 : 0].as<uint32_t>(); }
    PreprocessOut pp() const;
    FrameBuffers fb() const;
};

// NCCL communicator of a data-parallel rank (comm.cpp; NCCL is loaded at run time).
struct Comm;
struct CommDeleter {
    void operator()(Comm* c) const;
};
void nccl_unique_id(unsigned char out[128]);  // ncclGetUniqueId
int nccl_version();

class Engine {
public:
    Engine(int device, cudaStream_t stream);
    ~Engine();
    Engine(const Engine&) = delete;
    Engine& operator=(const Engine&) = delete;

    void upload(const HostCloud& cloud);
    HostCloud download();
    void set_active_sh_degree(int d);

    Frame* render(const double pose12[12], int W, int H, const double bg[3]);
    // bin_to_tiles + blend_forward over host SplatProjection records (kSplatPlanes FP64 planes of
    // n, kernels.h): K2 bins and sorts them by (depth, slot) unless a tile grid is supplied
    // (ranges per tile into `slots`, each a record index), then K3 blends.
    Frame* render_projected(const double* planes, size_t n, int W, int H, const double bg[3],
                            const std::vector<uint2>* ranges = nullptr, const std::vector<uint32_t>* slots = nullptr);
    // First use of a frame's results: waits for its instance count and re-renders it in the rare
    // case of an instance-buffer overflow or a long run of equal FP32 depth keys.
    void validate(Frame* f);
    // cov (3 planes) and camera-space centre t (3 planes) of the frame's Gaussians (n each,
    // zeros when culled): the SplatProjection fields K1 does not store.
    void projection_detail(Frame* f, std::vector<double>& out);
    void release(Frame* f);
    void backward(Frame* f, const float* d_image_planar_dev, bool accumulate);
    // Optional deterministic backward (gradients.cpp:94-169's fixed-order reduction): K4a without
    // atomics, per-instance partials reduced per Gaussian in a fixed order — gradients bit-identical
    // run to run, at roughly twice K4a's cost. Off by default.
    void set_deterministic(bool on) { deterministic_ = on; }
    // Strict T-stop guard in K3 (common.cuh): the FP32 transmittance carries a rigorous error bound
    // instead of the fixed 2^-10 band — a verification mode (more FP64 replays, ~1.8x K3 time).
    void set_strict_guard(bool on) { strict_guard_ = on; }
    bool deterministic() const { return deterministic_; }
    // loss() of trainer.cpp:25-71 on the device: d_image into d_image_buffer(); the value is read
    // back only when want_value (one 32-byte read, synchronizes the stream).
    double loss(Frame* f, const float* gt_planar_dev, double lambda_ssim, double mask_bottom_fraction,
                bool want_value);
    double loss_value(const Frame* f, double mask_bottom_fraction);
    // Enqueue a copy of the loss sums {L1, SSIM r, g, b} into host memory (pinned, or the copy is
    // synchronous); valid once the stream has reached this point.
    void loss_sums_async(double* host);
    // The frame's colour as H x W x 3 doubles (Image layout, image.hpp:10-23) in host memory:
    // converted on the device, one D2H copy (full speed into pinned memory), synchronous.
    void image_hwc(Frame* f, double* host);
    // render + image_hwc with the host copy overlapped: K3 blends the frame in bands of tile rows
    // and each band is converted and copied to `host` (pinned) on a side stream while the next band
    // blends. Returns the frame (validated; its image is in `host`).
    Frame* render_hwc(const double pose12[12], int W, int H, const double bg[3], double* host);
    // The same conversion into a device buffer owned by the engine (valid until the next call).
    const double* image_hwc_device(Frame* f);
    // Adam over all planes, or over the flat element range [begin, begin + count) (multiples of 4;
    // a data-parallel rank's shard after a reduce-scatter of the gradients).
    void adam_step(const TrainHyper& h, double extent, long iteration, bool zero_grad, size_t begin = 0,
                   size_t count = ~size_t(0));
    // Gradients are tracked as "logically zero" after zero_grad / a consuming Adam step, so the next
    // backward stores instead of read-modify-writes; materialize_grads() writes the zeros when the
    // buffer itself is about to be read (download, external views, Adam without a backward).
    void zero_grad();
    void materialize_grads();
    bool grads_zero() const { return grads_zero_; }
    void reset_screen_stats();
    // Trainer construction / resume (trainer.cpp:313-332): GradientBuffer and DensifyStats start
    // from zero (screen statistics, d_screen, max radii, gradients); a fresh run (fresh = true)
    // also restarts Adam (moments zero, step 0), a resume keeps the loaded optimizer state.
    void begin_training(bool fresh);
    // Densification control (trainer.cpp:180-280): DensifyStats::observe of a rendered frame,
    // densify_and_prune with the reference's RNG stream std::mt19937_64(rng_seed), reset_opacity.
    void observe(Frame* f);
    EditSummary densify_and_prune(const DensifyArgs& a, unsigned long long rng_seed);
    void reset_opacity(double ceiling);
    // psnr (metrics.cpp:64-74) of a frame against a device planar FP32 image (synchronizes).
    double psnr(Frame* f, const float* gt_planar);
    // Adam moments as raw planes (planes x stride floats each) and the step counter.
    void read_adam(std::vector<float>& m, std::vector<float>& v);
    void write_adam(const std::vector<float>& m, const std::vector<float>& v, long step);
    void synchronize();

    // ---- multi-view data parallelism over NCCL (comm.cpp), one process (context) per GPU.
    // dp_init: ncclCommInitRank on this context's device. dp_step: in-place reduce-scatter of the
    // gradient planes, fused Adam on this rank's 1/world shard, in-place all-gather of the
    // parameters, all on the context stream (sharded optimizer; replicas stay bit-identical).
    // With a communicator, densify_and_prune first sums the screen statistics / maxes the radii
    // over ranks and gathers the Adam moments; read_adam (the OSPLADAM sidecar) gathers them too.
    void dp_init(int world, int rank, const unsigned char id[128]);
    int dp_world() const;
    int dp_rank() const;
    void dp_step(const TrainHyper& h, double extent, long iteration);
    void dp_gather_moments();
    void dp_reduce_stats();
    // CUDA-event timing per kernel family on the context stream, and per-pixel work counting.
    void set_profiling(bool timing, bool count_work);
    void profile_read(double* ms, long* launches, bool reset);

    // accessors
    cudaStream_t stream() const { return stream_; }
    int device() const { return device_; }
    size_t n() const { return n_; }
    // Bumped whenever the Gaussian set is replaced (upload, densify): frames of an older
    // generation no longer describe the cloud (StateMismatch).
    unsigned long generation() const { return generation_; }
    size_t stride() const { return stride_; }
    int planes() const { return planes_; }
    int sh_degree() const { return sh_degree_; }
    int active_sh_degree() const { return active_; }
    long adam_step_count() const { return adam_step_; }
    float* params() const { return params_.as<float>(); }
    float* grads() const { return grads_.as<float>(); }
    float* adam_m() const { return m_.as<float>(); }
    float* adam_v() const { return v_.as<float>(); }
    float2* d_screen() const { return d_screen_.as<float2>(); }
    double* norm_sum() const { return norm_sum_.as<double>(); }
    int* hits() const { return hits_.as<int>(); }
    float* max_radius() const { return max_radius_.as<float>(); }
    float* d_image_buffer(size_t pixels);
    float* gt_buffer(size_t pixels);
    // Host target upload on a side stream (overlaps the render): upload -> wait_target() on the
    // main stream before the first consumer -> release_target() after the last consumer.
    const float* upload_target_async(const float* host, size_t pixels);
    void wait_target();
    void release_target();

private:
    int device_;
    cudaStream_t stream_;
    bool own_stream_;
    size_t n_ = 0, stride_ = 0;
    unsigned long generation_ = 0;
    int planes_ = 0, sh_degree_ = 0, active_ = 0;
    long adam_step_ = 0;
    DevBuf scratch_;
    DevBuf params_, grads_, m_, v_, acc_, d_screen_, norm_sum_, hits_, max_radius_, loss_sum_, d_image_, gt_,
        ssim_planes_, hwc_;
    // densify_and_prune scratch and the spare parameter / moment planes it writes into
    DevBuf dz_code_, dz_rank_, dz_ws_, dz_csrc_, dz_ssrc_, dz_normals_, dz_keep_, dz_dest_, spare_p_, spare_m_, spare_v_;
    void reset_per_gaussian_state();
    void render_into(Frame* f);
    void grow_instances(Frame* f, uint32_t M);  // zero gradients' screen stats, d_screen, max radius (GradientBuffer::resize)
    double last_lambda_ = 0.0;
    bool grads_zero_ = true;
    bool deterministic_ = false;
    bool strict_guard_ = false;
    std::unique_ptr<Comm, CommDeleter> comm_;
    bool moments_sharded_ = false;  // Adam moments outside this rank's shard are stale
    size_t dp_shard(size_t* begin) const;
    DevBuf det_inst_, det_rank_;
    std::vector<std::unique_ptr<Frame>> pool_;
    std::vector<Frame*> free_;
    cudaStream_t copy_stream_ = nullptr;
    // render_hwc: the host image of the frame being rendered (nullptr otherwise), its D2H stream and
    // band events; renders_ counts render_into calls (a validate() re-render is detected by it)
    double* hwc_host_ = nullptr;
    cudaStream_t d2h_stream_ = nullptr;
    std::vector<cudaEvent_t> band_ev_;
    unsigned long renders_ = 0;
    cudaEvent_t target_ready_ = nullptr, target_free_ = nullptr;

    // profiler
    struct Ev {
        int k;
        cudaEvent_t a, b;
    };
    bool timing_ = false, count_work_ = false;
    std::vector<Ev> pending_;
    std::vector<cudaEvent_t> events_;
    double prof_ms_[kKernelCount] = {};
    long prof_n_[kKernelCount] = {};
    cudaEvent_t ev_get();
    void collect();

public:
    // RAII span: records a start/stop event pair around a kernel family when timing is on.
    struct Span {
        Engine& e;
        int k;
        cudaEvent_t a = nullptr;
        Span(Engine& eng, int kind);
        ~Span();
    };
};

// RAII device guard.
struct DeviceGuard {
    int prev = 0;
    explicit DeviceGuard(int dev);
    ~DeviceGuard();
};

}  // namespace osb
