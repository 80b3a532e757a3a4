// trainer.cpp — Trainer::run on the device (proj/src/trainer.cpp:284-392) and the optimizer-state
// sidecar (proj/src/dataio.cpp:455-527).
//
// Every iteration is the reference's: pick_view (per-epoch Fisher-Yates shuffle seeded with
// mix64(seed ^ mix64(epoch))), SH warm-up, render -> loss -> backward (overwrite) -> observe,
// densify_and_prune every densify_interval up to densify_until with the rng
// mix64(seed ^ mix64(0x5eed + j)) (radius pruning after the first opacity reset), reset_opacity
// every opacity_reset_interval, and Adam unless the iteration densified. The whole iteration is
// device-resident (targets live in HBM); the stream is synchronised once per render (the instance
// count) and on log / densify iterations.
#include "trainer.h"

#include <cmath>
#include <cstdint>
#include <cstring>
#include <fstream>
#include <limits>
#include <random>
#include <stdexcept>

namespace osb {

unsigned long long mix64(unsigned long long x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

void TrainSettings::validate() const {
    if (lambda_ssim < 0.0 || lambda_ssim > 1.0) throw std::invalid_argument("ValidationError: lambda_ssim must be in [0, 1]");
    if (iterations < 0) throw std::invalid_argument("ValidationError: iterations must be >= 0");
    if (densify_interval <= 0 || opacity_reset_interval <= 0 || sh_warmup_interval <= 0)
        throw std::invalid_argument("ValidationError: intervals must be positive");
    if (densify_grad_threshold <= 0.0 || scale_split_threshold <= 0.0 || split_factor <= 0.0 || prune_opacity <= 0.0 ||
        prune_scale_world <= 0.0 || prune_radius_px <= 0.0)
        throw std::invalid_argument("ValidationError: densification thresholds must be positive");
    if (mask_bottom_fraction < 0.0 || mask_bottom_fraction >= 1.0)
        throw std::invalid_argument("ValidationError: mask_bottom_fraction must be in [0, 1)");
    if (sh_degree < 0 || sh_degree > 3) throw std::invalid_argument("ValidationError: sh_degree must be in 0..3");
}

DensifyArgs TrainSettings::densify_args(double extent, bool radius_active) const {
    DensifyArgs a;
    a.grad_threshold = densify_grad_threshold;
    a.split_scale = scale_split_threshold * extent;
    a.log_split = std::log(split_factor);
    a.prune_opacity = prune_opacity;
    a.prune_scale = prune_scale_world * extent;
    a.prune_radius = prune_radius_px;
    a.radius_active = radius_active ? 1 : 0;
    return a;
}

double scene_extent(const std::vector<double>& poses12, const std::vector<double>& points) {
    auto bounding_radius = [](const std::vector<double>& xyz) {
        const size_t n = xyz.size() / 3;
        if (n == 0) return 0.0;
        double mean[3] = {0.0, 0.0, 0.0};
        for (size_t i = 0; i < n; ++i)
            for (int k = 0; k < 3; ++k) mean[k] += xyz[3 * i + k];
        for (int k = 0; k < 3; ++k) mean[k] *= 1.0 / static_cast<double>(n);
        double r = 0.0;
        for (size_t i = 0; i < n; ++i) {
            const double d[3] = {xyz[3 * i] - mean[0], xyz[3 * i + 1] - mean[1], xyz[3 * i + 2] - mean[2]};
            const double len = std::sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
            r = r > len ? r : len;
        }
        return r;
    };
    // Pose::center = -R^T t (camera.hpp:26)
    std::vector<double> centres;
    for (size_t v = 0; v + 12 <= poses12.size(); v += 12) {
        const double* R = &poses12[v];
        const double* t = &poses12[v + 9];
        for (int c = 0; c < 3; ++c) centres.push_back(-(R[c] * t[0] + R[3 + c] * t[1] + R[6 + c] * t[2]));
    }
    double r = bounding_radius(centres) * 1.1;
    if (r > 1e-9) return r;
    r = bounding_radius(points) * 1.1;
    return r > 1e-9 ? r : 1.0;
}

DeviceTrainer::DeviceTrainer(Engine& e, const TrainSettings& cfg, std::vector<double> poses12, const float* images,
                             int width, int height, std::vector<int> train_indices, std::vector<int> test_indices,
                             double extent)
    : e_(e), cfg_(cfg), poses_(std::move(poses12)), W_(width), H_(height), train_(std::move(train_indices)),
      test_(std::move(test_indices)), extent_(extent) {
    cfg_.validate();
    if (train_.empty()) throw std::invalid_argument("ValidationError: dataset has no training views");
    const size_t views = poses_.size() / 12;
    for (int v : train_)
        if (v < 0 || static_cast<size_t>(v) >= views) throw std::invalid_argument("train view index out of range");
    for (int v : test_)
        if (v < 0 || static_cast<size_t>(v) >= views) throw std::invalid_argument("test view index out of range");
    DeviceGuard g(e_.device());
    const size_t bytes = views * 3 * static_cast<size_t>(W_) * H_ * sizeof(float);
    images_.ensure(bytes);
    OSB_CUDA_CHECK(cudaMemcpyAsync(images_.as<float>(), images, bytes, cudaMemcpyHostToDevice, e_.stream()));
    OSB_CUDA_CHECK(cudaStreamSynchronize(e_.stream()));
}

int DeviceTrainer::pick_view(long iteration) { return view_at(iteration - 1); }

int DeviceTrainer::view_at(long s) {
    const long n = static_cast<long>(train_.size());
    const long epoch = s / n;
    if (epoch != epoch_) {
        epoch_ = epoch;
        order_ = train_;
        std::mt19937_64 rng(mix64(cfg_.seed ^ mix64(static_cast<std::uint64_t>(epoch))));
        for (size_t i = order_.size(); i > 1; --i) {
            const size_t j = rng() % i;
            std::swap(order_[i - 1], order_[j]);
        }
    }
    return order_[s % n];
}

void DeviceTrainer::run(long start_iteration, const std::function<void(const IterationReport&)>& hook) {
    DeviceGuard g(e_.device());
    // the reference Trainer sizes (zeroes) GradientBuffer / DensifyStats / AdamState in its
    // constructor (trainer.cpp:313-323); resume() then loads Adam (trainer.cpp:325-332)
    e_.begin_training(start_iteration == 0);
    iteration_ = start_iteration;
    epoch_ = -1;
    const int heldout = test_.empty() ? train_[0] : test_[0];
    const double nan = std::numeric_limits<double>::quiet_NaN();
    // data parallel (a communicator on the context, comm.cpp): iteration j trains a batch of `world`
    // views — entries (j - 1) world .. j world - 1 of the reference's view stream, entry
    // (j - 1) world + rank on this rank — then one exchange (sharded Adam, or the densify exchange);
    // at world 1 this is Trainer::run exactly
    const long world = e_.dp_world(), rank = e_.dp_rank();
    for (long j = iteration_ + 1; j <= cfg_.iterations; ++j) {
        iteration_ = j;
        const int view = view_at((j - 1) * world + rank);
        if (j % cfg_.sh_warmup_interval == 0) {
            const int d = e_.active_sh_degree() + 1;
            e_.set_active_sh_degree(d < e_.sh_degree() ? d : e_.sh_degree());
        }
        const bool log_now = cfg_.log_interval > 0 && (j % cfg_.log_interval == 0 || j == cfg_.iterations);
        Frame* f = e_.render(&poses_[12 * static_cast<size_t>(view)], W_, H_, cfg_.background);
        IterationReport rep;
        rep.iteration = j;
        try {
            e_.loss(f, image(view), cfg_.lambda_ssim, cfg_.mask_bottom_fraction, false);
            e_.backward(f, e_.d_image_buffer(static_cast<size_t>(W_) * H_), false);
            e_.observe(f);
            rep.loss = log_now ? e_.loss_value(f, cfg_.mask_bottom_fraction) : nan;
        } catch (...) {
            e_.release(f);
            throw;
        }
        e_.release(f);
        if (j <= cfg_.densify_until) {
            if (j % cfg_.densify_interval == 0) {
                const unsigned long long seed = mix64(cfg_.seed ^ mix64(0x5eedULL + static_cast<std::uint64_t>(j)));
                rep.edit = e_.densify_and_prune(cfg_.densify_args(extent_, j > cfg_.opacity_reset_interval), seed);
                rep.densified = true;
            }
            if (j % cfg_.opacity_reset_interval == 0) e_.reset_opacity(cfg_.opacity_reset_ceiling);
        }
        // the densification edit rebuilds the parameter arrays: this iteration's gradients no longer apply
        if (!rep.densified) {
            if (world > 1) e_.dp_step(cfg_.lr, extent_, j);
            else e_.adam_step(cfg_.lr, extent_, j, true);
        }
        rep.gaussians = e_.n();
        rep.logged = log_now;
        rep.heldout_psnr = nan;
        if (log_now) {
            Frame* h = e_.render(&poses_[12 * static_cast<size_t>(heldout)], W_, H_, cfg_.background);
            try {
                rep.heldout_psnr = e_.psnr(h, image(heldout));
            } catch (...) {
                e_.release(h);
                throw;
            }
            e_.release(h);
        }
        if (hook) hook(rep);
    }
}

// ------------------------------------------------------------------ optimizer-state sidecar

namespace {

constexpr char kStateMagic[8] = {'O', 'S', 'P', 'L', 'A', 'D', 'A', 'M'};
constexpr std::uint32_t kStateVersion = 1;

// Reference AdamState arrays (trainer.hpp:64-75) as (first plane, values per Gaussian) of the
// plane layout: position 3, SH 3*bc (basis-major, channel-minor = plane order), rotation 4,
// log-scale 3, opacity 1 — each array once for m and once for v, interleaved m, v, m, v...
struct Group {
    int first, count;
};

std::vector<Group> groups(int bc) {
    const Planes pl{bc};
    return {{0, 3}, {pl.sh(0, 0), 3 * bc}, {pl.rot(0), 4}, {pl.lscale(0), 3}, {pl.opacity(), 1}};
}

}  // namespace

void save_optimizer_state(Engine& e, long iteration, const std::string& path) {
    std::vector<float> m, v;
    e.read_adam(m, v);
    const size_t n = e.n(), stride = e.stride();
    const int bc = (e.sh_degree() + 1) * (e.sh_degree() + 1);
    std::ofstream out(path, std::ios::binary);
    if (!out) throw std::runtime_error("IoError: cannot write " + path);
    out.write(kStateMagic, 8);
    out.write(reinterpret_cast<const char*>(&kStateVersion), 4);
    const std::int64_t iter = iteration, step = e.adam_step_count();
    const std::int32_t bc32 = bc;
    out.write(reinterpret_cast<const char*>(&iter), 8);
    out.write(reinterpret_cast<const char*>(&step), 8);
    out.write(reinterpret_cast<const char*>(&bc32), 4);
    std::vector<double> buf;
    for (const Group& gr : groups(bc)) {
        for (const std::vector<float>* src : {&m, &v}) {
            buf.resize(n * gr.count);
            for (size_t i = 0; i < n; ++i)
                for (int k = 0; k < gr.count; ++k) buf[i * gr.count + k] = (*src)[(gr.first + k) * stride + i];
            const std::uint64_t cnt = buf.size();
            out.write(reinterpret_cast<const char*>(&cnt), 8);
            out.write(reinterpret_cast<const char*>(buf.data()), static_cast<std::streamsize>(cnt * 8));
        }
    }
    if (!out) throw std::runtime_error("IoError: cannot write " + path);
}

long load_optimizer_state(Engine& e, const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw std::runtime_error("IoError: cannot open " + path);
    char magic[8];
    if (!in.read(magic, 8) || std::memcmp(magic, kStateMagic, 8) != 0)
        throw std::runtime_error("ParseError: " + path + ": not an optimizer state file");
    std::uint32_t version = 0;
    in.read(reinterpret_cast<char*>(&version), 4);
    if (version != kStateVersion)
        throw std::runtime_error("VersionMismatch: " + path + ": state version " + std::to_string(version));
    std::int64_t iter = 0, step = 0;
    std::int32_t bc = 0;
    in.read(reinterpret_cast<char*>(&iter), 8);
    in.read(reinterpret_cast<char*>(&step), 8);
    in.read(reinterpret_cast<char*>(&bc), 4);
    const int ebc = (e.sh_degree() + 1) * (e.sh_degree() + 1);
    if (bc != ebc) throw std::runtime_error("ValidationError: " + path + ": basis count does not match the cloud");
    const size_t n = e.n(), stride = e.stride();
    std::vector<float> m(static_cast<size_t>(e.planes()) * stride, 0.0f), v(m.size(), 0.0f);
    std::vector<double> buf;
    for (const Group& gr : groups(bc)) {
        for (std::vector<float>* dst : {&m, &v}) {
            std::uint64_t cnt = 0;
            if (!in.read(reinterpret_cast<char*>(&cnt), 8)) throw std::runtime_error("ParseError: " + path + ": truncated state file");
            if (cnt != n * static_cast<std::uint64_t>(gr.count))
                throw std::runtime_error("ValidationError: " + path + ": state size does not match the cloud");
            buf.resize(cnt);
            if (!in.read(reinterpret_cast<char*>(buf.data()), static_cast<std::streamsize>(cnt * 8)))
                throw std::runtime_error("ParseError: " + path + ": truncated state file");
            for (size_t i = 0; i < n; ++i)
                for (int k = 0; k < gr.count; ++k) (*dst)[(gr.first + k) * stride + i] = static_cast<float>(buf[i * gr.count + k]);
        }
    }
    e.write_adam(m, v, static_cast<long>(step));
    return static_cast<long>(iter);
}

}  // namespace osb
