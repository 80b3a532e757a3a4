// trainer.h — the reconstruction loop on the device (Trainer::run, proj/src/trainer.cpp:284-392)
// and the optimizer-state sidecar (proj/src/dataio.cpp:455-527).
#pragma once

#include <functional>
#include <string>
#include <vector>

#include "engine.h"

namespace osb {

// TrainConfig (proj/include/omnisplat/trainer.hpp:19-51), reference defaults.
struct TrainSettings {
    double lambda_ssim = 0.2;
    long iterations = 7000, densify_until = 15000, densify_interval = 100, opacity_reset_interval = 3000;
    double densify_grad_threshold = 2e-4, scale_split_threshold = 0.01, split_factor = 1.6, prune_opacity = 0.005;
    double prune_scale_world = 0.1, prune_radius_px = 20.0, opacity_reset_ceiling = 0.01;
    TrainHyper lr;
    double mask_bottom_fraction = 0.0;
    int sh_degree = 3;
    long sh_warmup_interval = 1000;
    unsigned long long seed = 0;
    long checkpoint_interval = 0, log_interval = 100;
    double background[3] = {0.0, 0.0, 0.0};

    void validate() const;  // TrainConfig::validate (trainer.cpp:10-23); throws std::invalid_argument
    DensifyArgs densify_args(double extent, bool radius_active) const;
};

unsigned long long mix64(unsigned long long x);  // trainer.cpp:300-306

// Per-iteration report handed to the hook (IterationInfo, trainer.hpp:108-114). loss / psnr are
// only evaluated on log iterations (they synchronize the stream); NaN otherwise.
struct IterationReport {
    long iteration = 0;
    double loss = 0.0, heldout_psnr = 0.0;
    size_t gaussians = 0;
    bool logged = false, densified = false;
    EditSummary edit;
};

// Trainer over an in-memory view set: poses (12 doubles each: row-major world->camera rotation,
// translation) and planar FP32 images (3 planes of W*H per view), all views uploaded to HBM once.
// Starts from the context's current parameters and Adam state (Trainer::resume semantics).
class DeviceTrainer {
public:
    DeviceTrainer(Engine& e, const TrainSettings& cfg, std::vector<double> poses12, const float* images_planar,
                  int width, int height, std::vector<int> train_indices, std::vector<int> test_indices,
                  double scene_extent);
    int pick_view(long iteration);  // trainer.cpp:340-354
    int view_at(long stream_index);  // entry of the per-epoch shuffled view stream (0-based)
    long iteration() const { return iteration_; }
    double extent() const { return extent_; }
    // Runs iterations iteration()+1 .. cfg.iterations; hook(report) after every iteration.
    void run(long start_iteration, const std::function<void(const IterationReport&)>& hook);

private:
    Engine& e_;
    TrainSettings cfg_;
    std::vector<double> poses_;
    int W_, H_;
    std::vector<int> train_, test_;
    double extent_;
    long iteration_ = 0, epoch_ = -1;
    std::vector<int> order_;
    DevBuf images_;
    const float* image(int view) const { return images_.as<float>() + static_cast<size_t>(view) * 3 * W_ * H_; }
};

// scene_extent (trainer.cpp:282-298): 1.1 x bounding radius of the camera centres, else of the
// points, else 1.
double scene_extent(const std::vector<double>& poses12, const std::vector<double>& points_xyz);

// save/load_optimizer_state (dataio.cpp:479-527): "OSPLADAM" v1, iteration, step, basis count and
// the ten moment arrays in the reference AdamState layouts, as doubles.
void save_optimizer_state(Engine& e, long iteration, const std::string& path);
long load_optimizer_state(Engine& e, const std::string& path);  // returns the stored iteration

}  // namespace osb
