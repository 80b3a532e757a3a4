// capi.cpp — the C ABI (include/osplat.h): the reference osplat_* symbols for this path
// (proj/src/capi.cpp) plus the device-resident extension. Error mapping follows
// capi.cpp:41-81: typed errors -> osplat_status, "<ErrorCode>: message" in a thread-local
// buffer that is cleared on success.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <charconv>
#include <chrono>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <memory>
#include <mutex>
#include <sstream>
#include <string>
#include <vector>

#include "../../include/osplat.h"
#include "engine.h"
#include "trainer.h"

using osb::Engine;
using osb::HostCloud;

// The reference's GaussianCloud is read-shared during rendering: any number of host
// threads may call osplat_render on one const cloud at once. The device copy (render_cache) and
// its Engine (stream, frame pool, staging buffers) are created once under render_mu, and each
// render holds render_mu for its K1 -> K3 + copy-out, so concurrent callers are serialised on the
// cloud's stream instead of racing on the Engine.
struct osplat_cloud {
    HostCloud cloud;
    mutable std::shared_ptr<Engine> render_cache;  // device copy used by osplat_render
    mutable std::mutex render_mu;
};
// H x W x 3 doubles. Images from osplat_render live in page-locked buffers recycled through a
// small pool (no page faults, full-speed D2H); images built from host data use the heap.
struct osplat_image {
    int width = 0, height = 0;
    std::vector<double> data;
    double* pinned = nullptr;
    size_t pinned_bytes = 0;
    const double* px() const { return pinned ? pinned : data.data(); }
    ~osplat_image();
};

// EvalReport (eval.hpp:28-35)
struct osplat_report {
    struct View {
        int frame_index;
        double psnr, ssim;
    };
    std::vector<View> views;
    double mean_psnr = 0.0, mean_ssim = 0.0, seconds_per_frame = 0.0, fps = 0.0;
    std::string mode;
};

namespace {
struct PinnedPool {
    std::mutex mu;
    std::vector<std::pair<void*, size_t>> free;
};
PinnedPool& pinned_pool() {
    static PinnedPool* p = new PinnedPool;  // never destroyed: buffers may be freed after main returns
    return *p;
}
double* pinned_acquire(size_t bytes) {
    PinnedPool& pool = pinned_pool();
    {
        std::lock_guard<std::mutex> lock(pool.mu);
        for (size_t i = 0; i < pool.free.size(); ++i)
            if (pool.free[i].second == bytes) {
                void* p = pool.free[i].first;
                pool.free.erase(pool.free.begin() + static_cast<long>(i));
                return static_cast<double*>(p);
            }
    }
    void* p = nullptr;
    OSB_CUDA_CHECK(cudaMallocHost(&p, bytes));
    return static_cast<double*>(p);
}
void pinned_release(void* p, size_t bytes) {
    PinnedPool& pool = pinned_pool();
    std::lock_guard<std::mutex> lock(pool.mu);
    if (pool.free.size() < 4) {
        pool.free.emplace_back(p, bytes);
        return;
    }
    cudaFreeHost(p);
}
}  // namespace

osplat_image::~osplat_image() {
    if (pinned) pinned_release(pinned, pinned_bytes);
}
struct osplat_config {
    // TrainConfig (trainer.hpp:19-51) with the reference defaults
    double lambda_ssim = 0.2;
    long iterations = 7000, densify_until = 15000, densify_interval = 100, opacity_reset_interval = 3000;
    double densify_grad_threshold = 2e-4, scale_split_threshold = 0.01, split_factor = 1.6, prune_opacity = 0.005;
    double prune_scale_world = 0.1, prune_radius_px = 20.0, opacity_reset_ceiling = 0.01;
    double lr_position_init = 1.6e-4, lr_position_final = 1.6e-6, lr_sh_dc = 2.5e-3, lr_sh_rest = 2.5e-3 / 20.0;
    double lr_opacity = 5e-2, lr_scale = 5e-3, lr_rotation = 1e-3, mask_bottom_fraction = 0.0;
    int sh_degree = 3;
    long sh_warmup_interval = 1000;
    unsigned long long seed = 0;
    long checkpoint_interval = 0, log_interval = 100;
    double background[3] = {0.0, 0.0, 0.0};  // JSON-only in the reference (dataio.cpp:611-615)
};
struct osplat_gpu {
    std::shared_ptr<Engine> engine;
};
struct osplat_frame {
    std::shared_ptr<Engine> engine;
    osb::Frame* frame = nullptr;
    // frames of host projections: device slot -> projection index, and the records' gaussian ids
    std::vector<int32_t> slot_index, given_ids;
};

namespace {

// Reference ErrorCode subset used on this path (error.hpp:8-25) and its status mapping.
enum class Code { ValidationError, StateMismatch, DimensionMismatch, ParseError, UnsupportedFormat, MissingProperty,
                  VersionMismatch, IoError, InvalidArgument, EmptySplit };

struct ApiError : std::runtime_error {
    Code code;
    ApiError(Code c, const std::string& m) : std::runtime_error(m), code(c) {}
};

const char* code_name(Code c) {
    switch (c) {
        case Code::ValidationError: return "ValidationError";
        case Code::StateMismatch: return "StateMismatch";
        case Code::DimensionMismatch: return "DimensionMismatch";
        case Code::ParseError: return "ParseError";
        case Code::UnsupportedFormat: return "UnsupportedFormat";
        case Code::MissingProperty: return "MissingProperty";
        case Code::VersionMismatch: return "VersionMismatch";
        case Code::IoError: return "IoError";
        case Code::InvalidArgument: return "InvalidArgument";
        case Code::EmptySplit: return "EmptySplit";
    }
    return "Unknown";
}

osplat_status map_code(Code c) {  // capi.cpp:41-66
    switch (c) {
        case Code::ParseError:
        case Code::MissingProperty: return OSPLAT_ERR_PARSE;
        case Code::ValidationError:
        case Code::DimensionMismatch:
        case Code::EmptySplit:
        case Code::StateMismatch: return OSPLAT_ERR_VALIDATION;
        case Code::UnsupportedFormat:
        case Code::VersionMismatch: return OSPLAT_ERR_UNSUPPORTED;
        case Code::IoError: return OSPLAT_ERR_IO;
        case Code::InvalidArgument: return OSPLAT_ERR_INVALID_ARGUMENT;
    }
    return OSPLAT_ERR_RUNTIME;
}

thread_local std::string t_last_error;

template <typename Fn>
osplat_status wrap(Fn&& fn) {
    try {
        fn();
        t_last_error.clear();
        return OSPLAT_OK;
    } catch (const ApiError& e) {
        t_last_error = std::string(code_name(e.code)) + ": " + e.what();
        return map_code(e.code);
    } catch (const std::exception& e) {
        // engine / trainer errors carry the reference ErrorCode name as a "<Name>: " prefix
        const std::string m = e.what();
        static const Code all[] = {Code::ValidationError, Code::StateMismatch,     Code::DimensionMismatch,
                                   Code::ParseError,      Code::UnsupportedFormat, Code::MissingProperty,
                                   Code::VersionMismatch, Code::IoError,           Code::InvalidArgument};
        for (Code c : all) {
            const std::string prefix = std::string(code_name(c)) + ": ";
            if (m.compare(0, prefix.size(), prefix) == 0) {
                t_last_error = m;
                return map_code(c);
            }
        }
        if (dynamic_cast<const std::invalid_argument*>(&e)) {
            t_last_error = "InvalidArgument: " + m;
            return OSPLAT_ERR_INVALID_ARGUMENT;
        }
        t_last_error = m;
        return OSPLAT_ERR_RUNTIME;
    }
}

osplat_status invalid(const char* message) {
    t_last_error = message;
    return OSPLAT_ERR_INVALID_ARGUMENT;
}

// Row-major 4x4 -> pose (capi.cpp:88-95) and Pose::is_valid (camera.cpp:7-19).
void pose_from_rowmajor(const double t[16], double p12[12]) {
    for (int r = 0; r < 3; ++r) {
        for (int c = 0; c < 3; ++c) p12[r * 3 + c] = t[r * 4 + c];
        p12[9 + r] = t[r * 4 + 3];
    }
}

bool pose_is_valid(const double* w, double tol = 1e-6) {
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            double s = 0.0;
            for (int k = 0; k < 3; ++k) s += w[k * 3 + i] * w[k * 3 + j];
            double expect = i == j ? 1.0 : 0.0;
            if (std::abs(s - expect) > tol) return false;
        }
    double det = w[0] * (w[4] * w[8] - w[5] * w[7]) - w[1] * (w[3] * w[8] - w[5] * w[6]) +
                 w[2] * (w[3] * w[7] - w[4] * w[6]);
    return std::abs(det - 1.0) <= tol;
}

void checked_pose(const double t[16], double p12[12]) {
    pose_from_rowmajor(t, p12);
    if (!pose_is_valid(p12)) throw ApiError(Code::ValidationError, "pose rotation is not orthonormal");
}

int default_device() {
    const char* env = std::getenv("OSPLAT_DEVICE");
    return env ? std::atoi(env) : 0;
}

// ------------------------------------------------------------------ checkpoint PLY (dataio.cpp:347-453)

constexpr int kCheckpointVersion = 1;

void save_checkpoint(const HostCloud& c, const std::string& path) {
    const int bc = c.bc();
    std::ofstream out(path, std::ios::binary);
    if (!out) throw ApiError(Code::IoError, "cannot write " + path);
    out << "ply\nformat binary_little_endian 1.0\n";
    out << "comment format_version " << kCheckpointVersion << "\n";
    out << "comment sh_degree " << c.sh_degree << "\n";
    out << "element vertex " << c.n() << "\n";
    for (const char* p : {"x", "y", "z", "nx", "ny", "nz", "f_dc_0", "f_dc_1", "f_dc_2"})
        out << "property float " << p << "\n";
    for (int i = 0; i < (bc - 1) * 3; ++i) out << "property float f_rest_" << i << "\n";
    out << "property float opacity\n";
    for (int i = 0; i < 3; ++i) out << "property float scale_" << i << "\n";
    for (int i = 0; i < 4; ++i) out << "property float rot_" << i << "\n";
    out << "end_header\n";
    std::vector<float> row;
    for (size_t i = 0; i < c.n(); ++i) {
        row.clear();
        for (int k = 0; k < 3; ++k) row.push_back(static_cast<float>(c.positions[3 * i + k]));
        for (int k = 0; k < 3; ++k) row.push_back(0.0f);
        const double* sh = &c.sh[i * bc * 3];
        for (int ch = 0; ch < 3; ++ch) row.push_back(static_cast<float>(sh[ch]));
        for (int ch = 0; ch < 3; ++ch)  // f_rest channel-major (dataio.cpp:374-376)
            for (int j = 1; j < bc; ++j) row.push_back(static_cast<float>(sh[j * 3 + ch]));
        row.push_back(static_cast<float>(c.opacity[i]));
        for (int k = 0; k < 3; ++k) row.push_back(static_cast<float>(c.log_scales[3 * i + k]));
        for (int k = 0; k < 4; ++k) row.push_back(static_cast<float>(c.rotations[4 * i + k]));
        out.write(reinterpret_cast<const char*>(row.data()), static_cast<std::streamsize>(row.size() * 4));
    }
    if (!out) throw ApiError(Code::IoError, "write failed for " + path);
}

HostCloud load_checkpoint(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw ApiError(Code::IoError, "cannot open " + path);
    std::string line;
    std::getline(in, line);
    if (line != "ply") throw ApiError(Code::ParseError, path + ": not a PLY file");
    bool binary_le = false;
    size_t count = 0;
    int sh_degree = -1;
    std::vector<std::string> props;
    while (std::getline(in, line)) {
        if (!line.empty() && line.back() == '\r') line.pop_back();
        std::istringstream ls(line);
        std::string key;
        ls >> key;
        if (key == "format") {
            std::string fmt;
            ls >> fmt;
            binary_le = fmt == "binary_little_endian";
            if (!binary_le) throw ApiError(Code::UnsupportedFormat, path + ": only binary_little_endian checkpoints");
        } else if (key == "comment") {
            std::string k2;
            ls >> k2;
            if (k2 == "format_version") {
                int v = -1;
                ls >> v;
                if (v != kCheckpointVersion)
                    throw ApiError(Code::VersionMismatch, path + ": checkpoint format version " + std::to_string(v));
            } else if (k2 == "sh_degree") {
                ls >> sh_degree;
            }
        } else if (key == "element") {
            std::string name;
            ls >> name >> count;
            if (name != "vertex") throw ApiError(Code::UnsupportedFormat, path + ": unexpected element " + name);
        } else if (key == "property") {
            std::string type, name;
            ls >> type >> name;
            if (type != "float" && type != "float32")
                throw ApiError(Code::UnsupportedFormat, path + ": property " + name + " is not float32");
            props.push_back(name);
        } else if (key == "end_header") {
            break;
        }
    }
    if (!binary_le) throw ApiError(Code::ParseError, path + ": missing format line");
    auto find = [&](const std::string& n) -> int {
        for (size_t i = 0; i < props.size(); ++i)
            if (props[i] == n) return static_cast<int>(i);
        return -1;
    };
    int rest = 0;
    while (find("f_rest_" + std::to_string(rest)) >= 0) ++rest;
    if (rest % 3 != 0) throw ApiError(Code::ParseError, path + ": f_rest count not divisible by 3");
    const int bc_rest = rest / 3 + 1;
    if (sh_degree < 0) {
        int d = 0;
        while ((d + 1) * (d + 1) < bc_rest) ++d;
        sh_degree = d;
    }
    const int bc = (sh_degree + 1) * (sh_degree + 1);
    if (bc != bc_rest) throw ApiError(Code::ParseError, path + ": sh_degree does not match f_rest count");
    for (const char* r : {"x", "y", "z", "f_dc_0", "f_dc_1", "f_dc_2", "opacity", "scale_0", "scale_1", "scale_2",
                          "rot_0", "rot_1", "rot_2", "rot_3"})
        if (find(r) < 0) throw ApiError(Code::MissingProperty, path + ": missing property " + r);
    std::vector<float> data(count * props.size());
    if (!in.read(reinterpret_cast<char*>(data.data()), static_cast<std::streamsize>(data.size() * 4)))
        throw ApiError(Code::ParseError, path + ": truncated vertex data");
    HostCloud c;
    c.sh_degree = sh_degree;
    c.active_sh_degree = sh_degree;
    c.positions.resize(count * 3);
    c.sh.resize(count * bc * 3);
    c.rotations.resize(count * 4);
    c.log_scales.resize(count * 3);
    c.opacity.resize(count);
    const size_t np = props.size();
    auto col = [&](const std::string& n, size_t i) { return static_cast<double>(data[i * np + find(n)]); };
    for (size_t i = 0; i < count; ++i) {
        c.positions[3 * i] = col("x", i);
        c.positions[3 * i + 1] = col("y", i);
        c.positions[3 * i + 2] = col("z", i);
        for (int ch = 0; ch < 3; ++ch) c.sh[i * bc * 3 + ch] = col("f_dc_" + std::to_string(ch), i);
        for (int ch = 0; ch < 3; ++ch)
            for (int j = 1; j < bc; ++j)
                c.sh[(i * bc + j) * 3 + ch] = col("f_rest_" + std::to_string(ch * (bc - 1) + (j - 1)), i);
        c.opacity[i] = col("opacity", i);
        for (int k = 0; k < 3; ++k) c.log_scales[3 * i + k] = col("scale_" + std::to_string(k), i);
        for (int k = 0; k < 4; ++k) c.rotations[4 * i + k] = col("rot_" + std::to_string(k), i);
    }
    return c;
}

void set_config_field(osplat_config& c, const std::string& key, const std::string& value) {
    auto as_double = [&] { return std::stod(value); };
    auto as_long = [&] { return std::stol(value); };
    try {
        if (key == "lambda_ssim") c.lambda_ssim = as_double();
        else if (key == "iterations") c.iterations = as_long();
        else if (key == "densify_until") c.densify_until = as_long();
        else if (key == "densify_interval") c.densify_interval = as_long();
        else if (key == "opacity_reset_interval") c.opacity_reset_interval = as_long();
        else if (key == "densify_grad_threshold") c.densify_grad_threshold = as_double();
        else if (key == "scale_split_threshold") c.scale_split_threshold = as_double();
        else if (key == "split_factor") c.split_factor = as_double();
        else if (key == "prune_opacity") c.prune_opacity = as_double();
        else if (key == "prune_scale_world") c.prune_scale_world = as_double();
        else if (key == "prune_radius_px") c.prune_radius_px = as_double();
        else if (key == "opacity_reset_ceiling") c.opacity_reset_ceiling = as_double();
        else if (key == "lr_position_init") c.lr_position_init = as_double();
        else if (key == "lr_position_final") c.lr_position_final = as_double();
        else if (key == "lr_sh_dc") c.lr_sh_dc = as_double();
        else if (key == "lr_sh_rest") c.lr_sh_rest = as_double();
        else if (key == "lr_opacity") c.lr_opacity = as_double();
        else if (key == "lr_scale") c.lr_scale = as_double();
        else if (key == "lr_rotation") c.lr_rotation = as_double();
        else if (key == "mask_bottom_fraction") c.mask_bottom_fraction = as_double();
        else if (key == "sh_degree") c.sh_degree = static_cast<int>(as_long());
        else if (key == "sh_warmup_interval") c.sh_warmup_interval = as_long();
        else if (key == "seed") c.seed = std::stoull(value);
        else if (key == "checkpoint_interval") c.checkpoint_interval = as_long();
        else if (key == "log_interval") c.log_interval = as_long();
        else throw ApiError(Code::ParseError, "unknown config key: " + key);
    } catch (const std::invalid_argument&) {
        throw ApiError(Code::ParseError, "config value for " + key + " is not a number: " + value);
    } catch (const std::out_of_range&) {
        throw ApiError(Code::ParseError, "config value for " + key + " is out of range: " + value);
    }
}

osb::TrainHyper hyper_from(const osplat_config* c) {
    osb::TrainHyper h;
    if (!c) return h;
    h.iterations = c->iterations;
    h.lr_position_init = c->lr_position_init;
    h.lr_position_final = c->lr_position_final;
    h.lr_sh_dc = c->lr_sh_dc;
    h.lr_sh_rest = c->lr_sh_rest;
    h.lr_opacity = c->lr_opacity;
    h.lr_scale = c->lr_scale;
    h.lr_rotation = c->lr_rotation;
    return h;
}

void check_dims(int w, int h) {
    if (w < 2 || h < 2) throw ApiError(Code::InvalidArgument, "image size must be >= 2x2");
    if (static_cast<long long>(w) * h > (1ll << 30)) throw ApiError(Code::InvalidArgument, "image too large");
}

osb::TrainSettings settings_from(const osplat_config* c) {
    const osplat_config d{};
    if (!c) c = &d;
    osb::TrainSettings t;
    t.lambda_ssim = c->lambda_ssim;
    t.iterations = c->iterations;
    t.densify_until = c->densify_until;
    t.densify_interval = c->densify_interval;
    t.opacity_reset_interval = c->opacity_reset_interval;
    t.densify_grad_threshold = c->densify_grad_threshold;
    t.scale_split_threshold = c->scale_split_threshold;
    t.split_factor = c->split_factor;
    t.prune_opacity = c->prune_opacity;
    t.prune_scale_world = c->prune_scale_world;
    t.prune_radius_px = c->prune_radius_px;
    t.opacity_reset_ceiling = c->opacity_reset_ceiling;
    t.lr = hyper_from(c);
    t.mask_bottom_fraction = c->mask_bottom_fraction;
    t.sh_degree = c->sh_degree;
    t.sh_warmup_interval = c->sh_warmup_interval;
    t.seed = c->seed;
    t.checkpoint_interval = c->checkpoint_interval;
    t.log_interval = c->log_interval;
    for (int k = 0; k < 3; ++k) t.background[k] = c->background[k];
    // TrainConfig::validate (trainer.cpp:10-23) with the reference's error code
    try {
        t.validate();
    } catch (const std::invalid_argument& e) {
        std::string m = e.what();
        const std::string prefix = "ValidationError: ";
        if (m.compare(0, prefix.size(), prefix) == 0) m = m.substr(prefix.size());
        throw ApiError(Code::ValidationError, m);
    }
    return t;
}

// nlohmann::json's number format (shortest round-trip digits; fixed notation for decimal exponents
// in (-4, 15], ".0" on integral values, else d.ddde+XX) so metrics.jsonl matches the reference's
// append_metrics_line (dataio.cpp:559-570) byte for byte.
std::string json_number(double v) {
    if (!std::isfinite(v)) return "null";
    if (v == 0.0) return std::signbit(v) ? "-0.0" : "0.0";
    char buf[64];
    auto r = std::to_chars(buf, buf + sizeof(buf), v, std::chars_format::scientific);
    std::string sci(buf, r.ptr);
    std::string out;
    if (sci[0] == '-') {
        out = "-";
        sci = sci.substr(1);
    }
    const size_t epos = sci.find('e');
    std::string digits = sci.substr(0, epos);
    digits.erase(std::remove(digits.begin(), digits.end(), '.'), digits.end());
    const int exp10 = std::stoi(sci.substr(epos + 1));
    const int k = static_cast<int>(digits.size());
    const int n = exp10 + 1;  // position of the decimal point
    if (k <= n && n <= 15) return out + digits + std::string(n - k, '0') + ".0";
    if (0 < n && n <= 15) return out + digits.substr(0, n) + "." + digits.substr(n);
    if (-4 < n && n <= 0) return out + "0." + std::string(-n, '0') + digits;
    std::string m = k == 1 ? digits : digits.substr(0, 1) + "." + digits.substr(1);
    const int e = n - 1;
    char eb[16];
    std::snprintf(eb, sizeof(eb), "e%c%02d", e < 0 ? '-' : '+', e < 0 ? -e : e);
    return out + m + eb;
}

}  // namespace

extern "C" {

const char* osplat_version(void) { return "0.1.0"; }
const char* osplat_last_error(void) { return t_last_error.c_str(); }
void osplat_set_threads(int) {}

osplat_status osplat_cloud_load(const char* path, osplat_cloud** out) {
    if (!path || !out) return invalid("osplat_cloud_load: null argument");
    return wrap([&] { *out = new osplat_cloud{load_checkpoint(path), nullptr, {}}; });
}

osplat_status osplat_cloud_save(const osplat_cloud* cloud, const char* path) {
    if (!cloud || !path) return invalid("osplat_cloud_save: null argument");
    return wrap([&] { save_checkpoint(cloud->cloud, path); });
}

size_t osplat_cloud_count(const osplat_cloud* cloud) { return cloud ? cloud->cloud.n() : 0; }
void osplat_cloud_free(osplat_cloud* cloud) { delete cloud; }

osplat_status osplat_cloud_create(size_t n, int sh_degree, int active, const double* positions, const double* sh,
                                  const double* rotations, const double* log_scales, const double* opacity,
                                  osplat_cloud** out) {
    if (!out || (n > 0 && (!positions || !sh || !rotations || !log_scales || !opacity)))
        return invalid("osplat_cloud_create: null argument");
    if (sh_degree < 0 || sh_degree > 3) return invalid("osplat_cloud_create: sh_degree must be in 0..3");
    return wrap([&] {
        auto* c = new osplat_cloud;
        HostCloud& h = c->cloud;
        h.sh_degree = sh_degree;
        h.active_sh_degree = active < 0 ? 0 : (active > sh_degree ? sh_degree : active);
        const size_t bc = static_cast<size_t>(h.bc());
        h.positions.assign(positions, positions + 3 * n);
        h.sh.assign(sh, sh + 3 * bc * n);
        h.rotations.assign(rotations, rotations + 4 * n);
        h.log_scales.assign(log_scales, log_scales + 3 * n);
        h.opacity.assign(opacity, opacity + n);
        *out = c;
    });
}

osplat_status osplat_cloud_read(const osplat_cloud* cloud, double* positions, double* sh, double* rotations,
                                double* log_scales, double* opacity, int* sh_degree, int* active) {
    if (!cloud) return invalid("osplat_cloud_read: null cloud");
    const HostCloud& h = cloud->cloud;
    auto cp = [](const std::vector<double>& v, double* dst) {
        if (dst && !v.empty()) std::memcpy(dst, v.data(), v.size() * 8);
    };
    cp(h.positions, positions);
    cp(h.sh, sh);
    cp(h.rotations, rotations);
    cp(h.log_scales, log_scales);
    cp(h.opacity, opacity);
    if (sh_degree) *sh_degree = h.sh_degree;
    if (active) *active = h.active_sh_degree;
    t_last_error.clear();
    return OSPLAT_OK;
}

osplat_status osplat_config_create(osplat_config** out) {
    if (!out) return invalid("osplat_config_create: null argument");
    return wrap([&] { *out = new osplat_config{}; });
}

osplat_status osplat_config_set(osplat_config* config, const char* key, const char* value) {
    if (!config || !key || !value) return invalid("osplat_config_set: null argument");
    return wrap([&] { set_config_field(*config, key, value); });
}

void osplat_config_free(osplat_config* config) { delete config; }

osplat_status osplat_render(const osplat_cloud* cloud, const double transform_cw[16], int width, int height,
                            osplat_image** out) {
    if (!cloud || !transform_cw || !out) return invalid("osplat_render: null argument");
    if (width < 2 || height < 2) return invalid("osplat_render: image size must be >= 2x2");
    return wrap([&] {
        double p12[12];
        checked_pose(transform_cw, p12);
        std::lock_guard<std::mutex> lock(cloud->render_mu);
        if (!cloud->render_cache) {
            auto e = std::make_shared<Engine>(default_device(), nullptr);
            e->upload(cloud->cloud);
            cloud->render_cache = e;
        }
        Engine& e = *cloud->render_cache;
        const double bg[3] = {0.0, 0.0, 0.0};
        const size_t plane = static_cast<size_t>(width) * height;
        auto img = std::make_unique<osplat_image>();
        img->width = width;
        img->height = height;
        img->pinned_bytes = plane * 3 * sizeof(double);
        img->pinned = pinned_acquire(img->pinned_bytes);
        // FP32 planes -> H x W x 3 doubles on the device, copied to the pinned image band by band
        // while the rest of the frame blends
        osb::Frame* f = e.render_hwc(p12, width, height, bg, img->pinned);
        e.release(f);
        *out = img.release();
    });
}

int osplat_image_width(const osplat_image* image) { return image ? image->width : 0; }
int osplat_image_height(const osplat_image* image) { return image ? image->height : 0; }
const double* osplat_image_pixels(const osplat_image* image) { return image ? image->px() : nullptr; }
void osplat_image_free(osplat_image* image) { delete image; }

// capi.cpp:287-296 -> psnr (metrics.cpp:64-74, capped at 99) and ssim (metrics.cpp:76-79) in FP64
// on the device: both images are uploaded, three kernels (metrics.cu) reduce them, the four sums
// come back and the host finishes the two formulas exactly as the reference does.
osplat_status osplat_metrics(const osplat_image* a, const osplat_image* b, double* out_psnr, double* out_ssim) {
    if (!a || !b) return invalid("osplat_metrics: null argument");
    return wrap([&] {
        if (a->width != b->width || a->height != b->height)
            throw ApiError(Code::DimensionMismatch, "psnr: image sizes differ");
        const int W = a->width, H = a->height;
        const size_t px = static_cast<size_t>(W) * H;
        osb::DeviceGuard g(default_device());
        cudaStream_t s = nullptr;
        OSB_CUDA_CHECK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
        void* buf = nullptr;
        const size_t img_bytes = px * 3 * sizeof(double);
        const size_t bytes = 2 * img_bytes + px * 15 * sizeof(double) + 4 * sizeof(double);
        double sums[4] = {0, 0, 0, 0};
        cudaError_t err = cudaMallocAsync(&buf, bytes, s);
        if (err == cudaSuccess) {
            double* da = static_cast<double*>(buf);
            double* db = da + px * 3;
            double* maps = db + px * 3;
            double* dsum = maps + px * 15;
            cudaMemcpyAsync(da, a->px(), img_bytes, cudaMemcpyHostToDevice, s);
            cudaMemcpyAsync(db, b->px(), img_bytes, cudaMemcpyHostToDevice, s);
            osb::launch_metrics_f64(da, db, W, H, maps, dsum, s);
            cudaMemcpyAsync(sums, dsum, sizeof(sums), cudaMemcpyDeviceToHost, s);
            cudaFreeAsync(buf, s);
            err = cudaStreamSynchronize(s);
        }
        cudaStreamDestroy(s);
        OSB_CUDA_CHECK(err);
        const double n = static_cast<double>(px) * 3.0;
        const double mse = sums[0] / n;
        if (out_psnr) *out_psnr = mse <= 0.0 ? 99.0 : std::min(99.0, 10.0 * std::log10(1.0 / mse));
        if (out_ssim) {
            double total = 0.0;
            for (int c = 0; c < 3; ++c) total += sums[1 + c] / static_cast<double>(px);
            *out_ssim = total / 3.0;
        }
    });
}

// ------------------------------------------------------------------ device-resident extension

osplat_status osplat_gpu_create(int device, void* stream, const osplat_cloud* cloud, osplat_gpu** out) {
    if (!cloud || !out) return invalid("osplat_gpu_create: null argument");
    return wrap([&] {
        auto g = std::make_unique<osplat_gpu>();
        g->engine = std::make_shared<Engine>(device, static_cast<cudaStream_t>(stream));
        g->engine->upload(cloud->cloud);
        *out = g.release();
    });
}

void osplat_gpu_free(osplat_gpu* ctx) { delete ctx; }
size_t osplat_gpu_count(const osplat_gpu* ctx) { return ctx ? ctx->engine->n() : 0; }

osplat_status osplat_gpu_set_deterministic(osplat_gpu* ctx, int on) {
    if (!ctx) return invalid("osplat_gpu_set_deterministic: null context");
    ctx->engine->set_deterministic(on != 0);
    t_last_error.clear();
    return OSPLAT_OK;
}

osplat_status osplat_gpu_set_strict_guard(osplat_gpu* ctx, int on) {
    if (!ctx) return invalid("osplat_gpu_set_strict_guard: null context");
    ctx->engine->set_strict_guard(on != 0);
    t_last_error.clear();
    return OSPLAT_OK;
}

osplat_status osplat_gpu_set_active_sh_degree(osplat_gpu* ctx, int degree) {
    if (!ctx) return invalid("osplat_gpu_set_active_sh_degree: null context");
    return wrap([&] { ctx->engine->set_active_sh_degree(degree); });
}

osplat_status osplat_gpu_download(osplat_gpu* ctx, osplat_cloud** out) {
    if (!ctx || !out) return invalid("osplat_gpu_download: null argument");
    return wrap([&] { *out = new osplat_cloud{ctx->engine->download(), nullptr, {}}; });
}

osplat_status osplat_gpu_synchronize(osplat_gpu* ctx) {
    if (!ctx) return invalid("osplat_gpu_synchronize: null context");
    return wrap([&] { ctx->engine->synchronize(); });
}

osplat_status osplat_gpu_render(osplat_gpu* ctx, const double transform_cw[16], int width, int height,
                                const double background[3], osplat_frame** out) {
    if (!ctx || !transform_cw || !out) return invalid("osplat_gpu_render: null argument");
    return wrap([&] {
        check_dims(width, height);
        double p12[12];
        checked_pose(transform_cw, p12);
        const double zero[3] = {0, 0, 0};
        auto fr = std::make_unique<osplat_frame>();
        fr->engine = ctx->engine;
        fr->frame = ctx->engine->render(p12, width, height, background ? background : zero);
        *out = fr.release();
    });
}

void osplat_frame_free(osplat_frame* frame) {
    if (!frame) return;
    frame->engine->release(frame->frame);
    delete frame;
}

int osplat_frame_width(const osplat_frame* f) { return f ? f->frame->W : 0; }
int osplat_frame_height(const osplat_frame* f) { return f ? f->frame->H : 0; }

osplat_status osplat_frame_image(const osplat_frame* frame, double* rgb) {
    if (!frame || !rgb) return invalid("osplat_frame_image: null argument");
    return wrap([&] {
        frame->engine->image_hwc(frame->frame, rgb);
    });
}

osplat_status osplat_frame_pixels(const osplat_frame* frame, float* rgb, float* T, int* contrib, int* last) {
    if (!frame) return invalid("osplat_frame_pixels: null frame");
    return wrap([&] {
        frame->engine->validate(frame->frame);
        const osb::Frame& f = *frame->frame;
        osb::DeviceGuard g(frame->engine->device());
        cudaStream_t s = frame->engine->stream();
        const size_t plane = static_cast<size_t>(f.W) * f.H;
        std::vector<float> host;
        if (rgb) {
            host.resize(plane * 3);
            OSB_CUDA_CHECK(cudaMemcpyAsync(host.data(), f.rgb.as<float>(), plane * 12, cudaMemcpyDeviceToHost, s));
        }
        if (T) OSB_CUDA_CHECK(cudaMemcpyAsync(T, f.T.as<float>(), plane * 4, cudaMemcpyDeviceToHost, s));
        if (contrib) OSB_CUDA_CHECK(cudaMemcpyAsync(contrib, f.contrib.as<int>(), plane * 4, cudaMemcpyDeviceToHost, s));
        if (last) OSB_CUDA_CHECK(cudaMemcpyAsync(last, f.last.as<int>(), plane * 4, cudaMemcpyDeviceToHost, s));
        OSB_CUDA_CHECK(cudaStreamSynchronize(s));
        if (rgb)
            for (size_t i = 0; i < plane; ++i)
                for (int c = 0; c < 3; ++c) rgb[i * 3 + c] = host[c * plane + i];
    });
}

osplat_status osplat_frame_projections(const osplat_frame* frame, uint8_t* visible, double* p, double* conic,
                                       double* opacity, float* color, int32_t* rect, uint32_t* touched) {
    if (!frame) return invalid("osplat_frame_projections: null frame");
    return wrap([&] {
        frame->engine->validate(frame->frame);
        const osb::Frame& f = *frame->frame;
        osb::DeviceGuard g(frame->engine->device());
        cudaStream_t s = frame->engine->stream();
        const size_t n = static_cast<size_t>(f.n);
        std::vector<uint64_t> key(n);
        std::vector<double2> pxy(n);
        std::vector<double4> co(n);
        std::vector<osb::Splat32> sp(n);
        std::vector<int4> rc(n);
        std::vector<uint32_t> tc(n);
        if (n) {
            OSB_CUDA_CHECK(cudaMemcpyAsync(key.data(), f.depth_key.as<void>(), n * 8, cudaMemcpyDeviceToHost, s));
            OSB_CUDA_CHECK(cudaMemcpyAsync(pxy.data(), f.pxy.as<void>(), n * 16, cudaMemcpyDeviceToHost, s));
            OSB_CUDA_CHECK(cudaMemcpyAsync(co.data(), f.conic_o.as<void>(), n * 32, cudaMemcpyDeviceToHost, s));
            OSB_CUDA_CHECK(cudaMemcpyAsync(sp.data(), f.splat.as<void>(), n * sizeof(osb::Splat32),
                                           cudaMemcpyDeviceToHost, s));
            OSB_CUDA_CHECK(cudaMemcpyAsync(rc.data(), f.rect.as<void>(), n * 16, cudaMemcpyDeviceToHost, s));
            OSB_CUDA_CHECK(cudaMemcpyAsync(tc.data(), f.touched.as<void>(), n * 4, cudaMemcpyDeviceToHost, s));
            OSB_CUDA_CHECK(cudaStreamSynchronize(s));
        }
        for (size_t i = 0; i < n; ++i) {
            const bool vis = key[i] != ~0ull;
            if (visible) visible[i] = vis ? 1 : 0;
            if (p) { p[2 * i] = vis ? pxy[i].x : 0.0; p[2 * i + 1] = vis ? pxy[i].y : 0.0; }
            if (conic) {
                conic[3 * i] = vis ? co[i].x : 0.0;
                conic[3 * i + 1] = vis ? co[i].y : 0.0;
                conic[3 * i + 2] = vis ? co[i].z : 0.0;
            }
            if (opacity) opacity[i] = vis ? co[i].w : 0.0;
            if (color) {
                color[3 * i] = vis ? sp[i].r : 0.0f;
                color[3 * i + 1] = vis ? sp[i].g : 0.0f;
                color[3 * i + 2] = vis ? sp[i].bl : 0.0f;
            }
            if (rect) {
                rect[4 * i] = vis ? rc[i].x : 0;
                rect[4 * i + 1] = vis ? rc[i].y : 0;
                rect[4 * i + 2] = vis ? rc[i].z : 0;
                rect[4 * i + 3] = vis ? rc[i].w : 0;
            }
            if (touched) touched[i] = vis ? tc[i] : 0;
        }
    });
}

osplat_status osplat_frame_tiles(const osplat_frame* frame, int* tiles_x, int* tiles_y, size_t* instances,
                                 uint32_t* ranges, uint32_t* gaussian_ids) {
    if (!frame) return invalid("osplat_frame_tiles: null frame");
    return wrap([&] {
        frame->engine->validate(frame->frame);
        const osb::Frame& f = *frame->frame;
        osb::DeviceGuard g(frame->engine->device());
        cudaStream_t s = frame->engine->stream();
        if (tiles_x) *tiles_x = f.tiles_x;
        if (tiles_y) *tiles_y = f.tiles_y;
        if (instances) *instances = f.M;
        const size_t tiles = static_cast<size_t>(f.tiles_x) * f.tiles_y;
        if (ranges) OSB_CUDA_CHECK(cudaMemcpyAsync(ranges, f.ranges.as<void>(), tiles * 8, cudaMemcpyDeviceToHost, s));
        if (gaussian_ids && f.M)
            OSB_CUDA_CHECK(cudaMemcpyAsync(gaussian_ids, f.inst_gid(), static_cast<size_t>(f.M) * 4,
                                           cudaMemcpyDeviceToHost, s));
        OSB_CUDA_CHECK(cudaStreamSynchronize(s));
        if (gaussian_ids && !frame->slot_index.empty())  // projection indices, like TileGrid
            for (size_t i = 0; i < f.M; ++i) gaussian_ids[i] = static_cast<uint32_t>(frame->slot_index[gaussian_ids[i]]);
    });
}

osplat_status osplat_gpu_upload(osplat_gpu* ctx, const osplat_cloud* cloud) {
    if (!ctx || !cloud) return invalid("osplat_gpu_upload: null argument");
    return wrap([&] { ctx->engine->upload(cloud->cloud); });
}

osplat_status osplat_gpu_render_projected(osplat_gpu* ctx, size_t count, const int32_t* gaussian_id, const double* p,
                                          const double* cov, const double* conic, const double* radius,
                                          const double* depth, const double* color, const double* alpha_base,
                                          int width, int height, const double background[3],
                                          const uint32_t* tile_offsets, const int32_t* tile_entries,
                                          osplat_frame** out) {
    if (!ctx || !out) return invalid("osplat_gpu_render_projected: null argument");
    if (count && (!p || !cov || !conic || !radius || !depth || !color || !alpha_base))
        return invalid("osplat_gpu_render_projected: null projection array");
    return wrap([&] {
        check_dims(width, height);
        if (count > static_cast<size_t>(INT32_MAX / osb::kSplatPlanes))
            throw ApiError(Code::InvalidArgument, "too many projections");
        for (size_t i = 0; i < count; ++i) {
            if (!std::isfinite(depth[i]) || depth[i] < 0.0)
                throw ApiError(Code::InvalidArgument, "projection depth must be finite and >= 0");
            if (!std::isfinite(p[2 * i]) || !std::isfinite(p[2 * i + 1]) || !std::isfinite(radius[i]) ||
                radius[i] < 0.0 || radius[i] > 1e9)
                throw ApiError(Code::InvalidArgument, "projection centre / radius out of range");
        }
        // device slots in (gaussian_id, index) order: K2's (depth, slot) order is then the
        // reference's (depth, gaussian_id) comparator (rasterizer.cpp:88-93)
        std::vector<int32_t> order(count);
        for (size_t i = 0; i < count; ++i) order[i] = static_cast<int32_t>(i);
        if (gaussian_id)
            std::stable_sort(order.begin(), order.end(),
                             [&](int32_t a, int32_t b) { return gaussian_id[a] < gaussian_id[b]; });
        std::vector<double> planes(count * osb::kSplatPlanes);
        auto put = [&](int plane, size_t slot, double v) { planes[plane * count + slot] = v; };
        for (size_t s = 0; s < count; ++s) {
            const size_t i = static_cast<size_t>(order[s]);
            put(0, s, p[2 * i]);
            put(1, s, p[2 * i + 1]);
            for (int k = 0; k < 3; ++k) {
                put(2 + k, s, cov[3 * i + k]);
                put(5 + k, s, conic[3 * i + k]);
                put(10 + k, s, color[3 * i + k]);
            }
            put(8, s, radius[i]);
            put(9, s, depth[i]);
            put(13, s, alpha_base[i]);
        }
        std::vector<uint2> ranges;
        std::vector<uint32_t> slots;
        if (tile_offsets) {
            const size_t tiles = static_cast<size_t>((width + 15) / 16) * ((height + 15) / 16);
            if (tile_offsets[0] != 0) throw ApiError(Code::InvalidArgument, "tile_offsets[0] must be 0");
            std::vector<uint32_t> slot_of(count);
            for (size_t s = 0; s < count; ++s) slot_of[order[s]] = static_cast<uint32_t>(s);
            ranges.resize(tiles);
            for (size_t t = 0; t < tiles; ++t) {
                if (tile_offsets[t + 1] < tile_offsets[t])
                    throw ApiError(Code::InvalidArgument, "tile_offsets must be non-decreasing");
                ranges[t] = make_uint2(tile_offsets[t], tile_offsets[t + 1]);
            }
            const size_t M = tile_offsets[tiles];
            if (M && !tile_entries) throw ApiError(Code::InvalidArgument, "null tile_entries");
            slots.resize(M);
            for (size_t e = 0; e < M; ++e) {
                if (tile_entries[e] < 0 || static_cast<size_t>(tile_entries[e]) >= count)
                    throw ApiError(Code::InvalidArgument, "tile entry out of range");
                slots[e] = slot_of[tile_entries[e]];
            }
        }
        const double zero[3] = {0, 0, 0};
        auto fr = std::make_unique<osplat_frame>();
        fr->engine = ctx->engine;
        fr->slot_index = order;
        if (fr->slot_index.empty()) fr->slot_index.push_back(0);  // marks a projection frame
        fr->given_ids.resize(count);
        for (size_t i = 0; i < count; ++i) fr->given_ids[i] = gaussian_id ? gaussian_id[i] : static_cast<int32_t>(i);
        fr->frame = ctx->engine->render_projected(planes.data(), count, width, height, background ? background : zero,
                                                  tile_offsets ? &ranges : nullptr, tile_offsets ? &slots : nullptr);
        *out = fr.release();
    });
}

osplat_status osplat_frame_splats(const osplat_frame* frame, size_t* count, int32_t* gaussian_id, double* p,
                                  double* cov, double* conic, double* radius, double* depth, double* color,
                                  double* alpha_base, double* t) {
    if (!frame || !count) return invalid("osplat_frame_splats: null argument");
    return wrap([&] {
        Engine& e = *frame->engine;
        e.validate(frame->frame);
        const osb::Frame& f = *frame->frame;
        osb::DeviceGuard g(e.device());
        cudaStream_t s = e.stream();
        const size_t n = static_cast<size_t>(f.n);
        if (f.projected) {  // the imported records, in projection order
            *count = n;
            std::vector<double> planes(n * osb::kSplatPlanes);
            if (n)
                OSB_CUDA_CHECK(cudaMemcpyAsync(planes.data(), f.import.as<double>(), planes.size() * 8,
                                               cudaMemcpyDeviceToHost, s));
            OSB_CUDA_CHECK(cudaStreamSynchronize(s));
            for (size_t slot = 0; slot < n; ++slot) {
                const size_t i = static_cast<size_t>(frame->slot_index[slot]);
                auto at = [&](int plane) { return planes[plane * n + slot]; };
                if (gaussian_id) gaussian_id[i] = frame->given_ids[i];
                for (int k = 0; k < 2; ++k) if (p) p[2 * i + k] = at(k);
                for (int k = 0; k < 3; ++k) {
                    if (cov) cov[3 * i + k] = at(2 + k);
                    if (conic) conic[3 * i + k] = at(5 + k);
                    if (color) color[3 * i + k] = at(10 + k);
                    if (t) t[3 * i + k] = 0.0;
                }
                if (radius) radius[i] = at(8);
                if (depth) depth[i] = at(9);
                if (alpha_base) alpha_base[i] = at(13);
            }
            return;
        }
        std::vector<uint64_t> key(n);
        std::vector<double2> pxy(n);
        std::vector<double4> co(n);
        std::vector<osb::Splat32> sp(n);
        std::vector<float> rad(n);
        if (n) {
            OSB_CUDA_CHECK(cudaMemcpyAsync(key.data(), f.depth_key.as<void>(), n * 8, cudaMemcpyDeviceToHost, s));
            OSB_CUDA_CHECK(cudaMemcpyAsync(pxy.data(), f.pxy.as<void>(), n * 16, cudaMemcpyDeviceToHost, s));
            OSB_CUDA_CHECK(cudaMemcpyAsync(co.data(), f.conic_o.as<void>(), n * 32, cudaMemcpyDeviceToHost, s));
            OSB_CUDA_CHECK(cudaMemcpyAsync(sp.data(), f.splat.as<void>(), n * sizeof(osb::Splat32),
                                           cudaMemcpyDeviceToHost, s));
            OSB_CUDA_CHECK(cudaMemcpyAsync(rad.data(), f.radius.as<void>(), n * 4, cudaMemcpyDeviceToHost, s));
        }
        OSB_CUDA_CHECK(cudaStreamSynchronize(s));
        std::vector<double> detail;
        const bool need_detail = cov || t;
        if (need_detail) e.projection_detail(frame->frame, detail);
        size_t v = 0;  // render()'s compaction: visible Gaussians in ascending id (rasterizer.cpp:165-168)
        for (size_t i = 0; i < n; ++i) {
            if (key[i] == ~0ull) continue;
            if (gaussian_id) gaussian_id[v] = static_cast<int32_t>(i);
            if (p) { p[2 * v] = pxy[i].x; p[2 * v + 1] = pxy[i].y; }
            if (conic) { conic[3 * v] = co[i].x; conic[3 * v + 1] = co[i].y; conic[3 * v + 2] = co[i].z; }
            if (alpha_base) alpha_base[v] = co[i].w;
            if (radius) radius[v] = rad[i];
            if (depth) { uint64_t b = key[i]; double d; std::memcpy(&d, &b, 8); depth[v] = d; }
            if (color) { color[3 * v] = sp[i].r; color[3 * v + 1] = sp[i].g; color[3 * v + 2] = sp[i].bl; }
            for (int k = 0; k < 3; ++k) {
                if (cov) cov[3 * v + k] = detail[k * n + i];
                if (t) t[3 * v + k] = detail[(3 + k) * n + i];
            }
            ++v;
        }
        *count = v;
    });
}

osplat_status osplat_frame_device(const osplat_frame* frame, osplat_frame_view* v) {
    if (!frame || !v) return invalid("osplat_frame_device: null argument");
    return wrap([&] {
        frame->engine->validate(frame->frame);
        const osb::Frame& f = *frame->frame;
        v->rgb = f.rgb.as<float>();
        v->transmittance = f.T.as<float>();
        v->contributors = f.contrib.as<int>();
        v->last_contrib = f.last.as<int>();
        v->width = f.W;
        v->height = f.H;
    });
}

osplat_status osplat_gpu_view_buffers(osplat_gpu* ctx, osplat_gpu_view* v) {
    if (!ctx || !v) return invalid("osplat_gpu_view_buffers: null argument");
    Engine& e = *ctx->engine;
    try {
        osb::DeviceGuard g(e.device());
        e.materialize_grads();  // the caller may read the gradient planes directly
    } catch (const std::exception& ex) {
        t_last_error = ex.what();
        return OSPLAT_ERR_RUNTIME;
    }
    v->params = e.params();
    v->grads = e.grads();
    v->adam_m = e.adam_m();
    v->adam_v = e.adam_v();
    v->d_screen = reinterpret_cast<float*>(e.d_screen());
    v->screen_norm_sum = e.norm_sum();
    v->screen_hits = e.hits();
    v->n = e.n();
    v->stride = e.stride();
    v->planes = e.planes();
    v->sh_degree = e.sh_degree();
    v->active_sh_degree = e.active_sh_degree();
    v->adam_step = e.adam_step_count();
    v->max_radius_px = e.max_radius();
    t_last_error.clear();
    return OSPLAT_OK;
}

static void validate_frame(osplat_gpu* ctx, const osplat_frame* frame) {
    if (frame->engine.get() != ctx->engine.get())
        throw ApiError(Code::StateMismatch, "frame was rendered by another context");
    if (static_cast<size_t>(frame->frame->n) != ctx->engine->n() || frame->frame->generation != ctx->engine->generation())
        throw ApiError(Code::StateMismatch, "render output does not match the given scene");
}

osplat_status osplat_gpu_backward(osplat_gpu* ctx, const osplat_frame* frame, const double* d_image, int accumulate) {
    if (!ctx || !frame || !d_image) return invalid("osplat_gpu_backward: null argument");
    return wrap([&] {
        validate_frame(ctx, frame);
        Engine& e = *ctx->engine;
        osb::DeviceGuard g(e.device());
        frame->engine->validate(frame->frame);
        const osb::Frame& f = *frame->frame;
        const size_t plane = static_cast<size_t>(f.W) * f.H;
        std::vector<float> planar(plane * 3);
        for (size_t i = 0; i < plane; ++i)
            for (int c = 0; c < 3; ++c) planar[c * plane + i] = static_cast<float>(d_image[i * 3 + c]);
        float* dev = e.d_image_buffer(plane);
        OSB_CUDA_CHECK(cudaMemcpyAsync(dev, planar.data(), plane * 12, cudaMemcpyHostToDevice, e.stream()));
        e.backward(frame->frame, dev, accumulate != 0);
        OSB_CUDA_CHECK(cudaStreamSynchronize(e.stream()));  // `planar` is pageable host memory
    });
}

osplat_status osplat_gpu_backward_device(osplat_gpu* ctx, const osplat_frame* frame, const float* d_image_planar,
                                         int accumulate) {
    if (!ctx || !frame || !d_image_planar) return invalid("osplat_gpu_backward_device: null argument");
    return wrap([&] {
        validate_frame(ctx, frame);
        ctx->engine->backward(frame->frame, d_image_planar, accumulate != 0);
    });
}

osplat_status osplat_gpu_gradients(osplat_gpu* ctx, double* d_position, double* d_sh, double* d_rotation,
                                   double* d_log_scale, double* d_opacity, double* d_screen, double* norm_sum,
                                   long* hits) {
    if (!ctx) return invalid("osplat_gpu_gradients: null context");
    return wrap([&] {
        Engine& e = *ctx->engine;
        osb::DeviceGuard g(e.device());
        const size_t n = e.n(), stride = e.stride();
        const int bc = (e.sh_degree() + 1) * (e.sh_degree() + 1);
        const osb::Planes pl{bc};
        e.materialize_grads();
        std::vector<float> G(static_cast<size_t>(e.planes()) * stride);
        std::vector<float2> ds(stride);
        std::vector<double> ns(stride);
        std::vector<int> hs(stride);
        cudaStream_t s = e.stream();
        OSB_CUDA_CHECK(cudaMemcpyAsync(G.data(), e.grads(), G.size() * 4, cudaMemcpyDeviceToHost, s));
        OSB_CUDA_CHECK(cudaMemcpyAsync(ds.data(), e.d_screen(), stride * 8, cudaMemcpyDeviceToHost, s));
        OSB_CUDA_CHECK(cudaMemcpyAsync(ns.data(), e.norm_sum(), stride * 8, cudaMemcpyDeviceToHost, s));
        OSB_CUDA_CHECK(cudaMemcpyAsync(hs.data(), e.hits(), stride * 4, cudaMemcpyDeviceToHost, s));
        OSB_CUDA_CHECK(cudaStreamSynchronize(s));
        for (size_t i = 0; i < n; ++i) {
            for (int k = 0; k < 3; ++k)
                if (d_position) d_position[3 * i + k] = G[k * stride + i];
            for (int b = 0; b < bc; ++b)
                for (int k = 0; k < 3; ++k)
                    if (d_sh) d_sh[(i * bc + b) * 3 + k] = G[pl.sh(b, k) * stride + i];
            for (int k = 0; k < 4; ++k)
                if (d_rotation) d_rotation[4 * i + k] = G[pl.rot(k) * stride + i];
            for (int k = 0; k < 3; ++k)
                if (d_log_scale) d_log_scale[3 * i + k] = G[pl.lscale(k) * stride + i];
            if (d_opacity) d_opacity[i] = G[pl.opacity() * stride + i];
            if (d_screen) { d_screen[2 * i] = ds[i].x; d_screen[2 * i + 1] = ds[i].y; }
            if (norm_sum) norm_sum[i] = ns[i];
            if (hits) hits[i] = hs[i];
        }
    });
}

osplat_status osplat_gpu_zero_grad(osplat_gpu* ctx) {
    if (!ctx) return invalid("osplat_gpu_zero_grad: null context");
    return wrap([&] { ctx->engine->zero_grad(); });
}

osplat_status osplat_gpu_reset_screen_stats(osplat_gpu* ctx) {
    if (!ctx) return invalid("osplat_gpu_reset_screen_stats: null context");
    return wrap([&] { ctx->engine->reset_screen_stats(); });
}

osplat_status osplat_gpu_observe(osplat_gpu* ctx, const osplat_frame* frame) {
    if (!ctx || !frame) return invalid("osplat_gpu_observe: null argument");
    return wrap([&] {
        validate_frame(ctx, frame);
        ctx->engine->observe(frame->frame);
    });
}

static osb::DensifyArgs densify_args(const osplat_config* c, double extent, int radius_active) {
    const osplat_config d{};
    if (!c) c = &d;
    if (c->densify_grad_threshold <= 0.0 || c->scale_split_threshold <= 0.0 || c->split_factor <= 0.0 ||
        c->prune_opacity <= 0.0 || c->prune_scale_world <= 0.0 || c->prune_radius_px <= 0.0)
        throw ApiError(Code::ValidationError, "densification thresholds must be positive");
    osb::DensifyArgs a;
    a.grad_threshold = c->densify_grad_threshold;
    a.split_scale = c->scale_split_threshold * extent;
    a.log_split = std::log(c->split_factor);
    a.prune_opacity = c->prune_opacity;
    a.prune_scale = c->prune_scale_world * extent;
    a.prune_radius = c->prune_radius_px;
    a.radius_active = radius_active != 0;
    return a;
}

osplat_status osplat_gpu_densify_and_prune(osplat_gpu* ctx, const osplat_config* config, double extent,
                                           unsigned long long rng_seed, int radius_prune_active,
                                           osplat_edit_summary* out) {
    if (!ctx) return invalid("osplat_gpu_densify_and_prune: null context");
    return wrap([&] {
        const osb::EditSummary e =
            ctx->engine->densify_and_prune(densify_args(config, extent, radius_prune_active), rng_seed);
        if (out) {
            out->cloned = e.cloned;
            out->split = e.split;
            out->pruned = e.pruned;
            out->final_count = e.final_count;
        }
    });
}

osplat_status osplat_gpu_reset_opacity(osplat_gpu* ctx, double ceiling) {
    if (!ctx) return invalid("osplat_gpu_reset_opacity: null context");
    if (!(ceiling > 0.0 && ceiling < 1.0)) return invalid("osplat_gpu_reset_opacity: ceiling must be in (0, 1)");
    return wrap([&] { ctx->engine->reset_opacity(ceiling); });
}

osplat_status osplat_gpu_max_radius(osplat_gpu* ctx, double* out) {
    if (!ctx || !out) return invalid("osplat_gpu_max_radius: null argument");
    return wrap([&] {
        Engine& e = *ctx->engine;
        osb::DeviceGuard g(e.device());
        std::vector<float> h(e.n());
        if (!h.empty())
            OSB_CUDA_CHECK(cudaMemcpyAsync(h.data(), e.max_radius(), h.size() * 4, cudaMemcpyDeviceToHost, e.stream()));
        OSB_CUDA_CHECK(cudaStreamSynchronize(e.stream()));
        for (size_t i = 0; i < h.size(); ++i) out[i] = h[i];
    });
}

unsigned long long osplat_mix64(unsigned long long x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

osplat_status osplat_image_create(int width, int height, const double* rgb, osplat_image** out) {
    if (!rgb || !out) return invalid("osplat_image_create: null argument");
    if (width < 1 || height < 1) return invalid("osplat_image_create: image size must be positive");
    return wrap([&] {
        auto img = std::make_unique<osplat_image>();
        img->width = width;
        img->height = height;
        img->data.assign(rgb, rgb + static_cast<size_t>(width) * height * 3);
        *out = img.release();
    });
}

osplat_status osplat_gpu_save_state(osplat_gpu* ctx, const char* path, long iteration) {
    if (!ctx || !path) return invalid("osplat_gpu_save_state: null argument");
    return wrap([&] { osb::save_optimizer_state(*ctx->engine, iteration, path); });
}

osplat_status osplat_gpu_load_state(osplat_gpu* ctx, const char* path, long* iteration) {
    if (!ctx || !path) return invalid("osplat_gpu_load_state: null argument");
    return wrap([&] {
        const long it = osb::load_optimizer_state(*ctx->engine, path);
        if (iteration) *iteration = it;
    });
}

osplat_status osplat_gpu_train(osplat_gpu* ctx, const osplat_config* config, size_t views,
                               const double* transforms_cw, const osplat_image* const* images, const uint8_t* is_test,
                               double scene_extent, long start_iteration, const char* output_dir,
                               osplat_progress_fn progress, void* user) {
    if (!ctx || !transforms_cw || !images) return invalid("osplat_gpu_train: null argument");
    if (views == 0) return invalid("osplat_gpu_train: no views");
    return wrap([&] {
        namespace fs = std::filesystem;
        const osb::TrainSettings cfg = settings_from(config);
        Engine& e = *ctx->engine;
        if (cfg.sh_degree != e.sh_degree())
            throw ApiError(Code::ValidationError, "config sh_degree does not match the cloud's");
        const int W = images[0] ? images[0]->width : 0, H = images[0] ? images[0]->height : 0;
        check_dims(W, H);
        std::vector<double> poses(12 * views);
        std::vector<int> train, test;
        const size_t plane = static_cast<size_t>(W) * H;
        std::vector<float> planar(views * 3 * plane);
        for (size_t v = 0; v < views; ++v) {
            checked_pose(transforms_cw + 16 * v, &poses[12 * v]);
            const osplat_image* im = images[v];
            if (!im) throw ApiError(Code::InvalidArgument, "null image");
            if (im->width != W || im->height != H)
                throw ApiError(Code::DimensionMismatch, "training images differ in size");
            float* dst = planar.data() + v * 3 * plane;
            for (size_t i = 0; i < plane; ++i)
                for (int c = 0; c < 3; ++c) dst[c * plane + i] = static_cast<float>(im->px()[3 * i + c]);
            (is_test && is_test[v] ? test : train).push_back(static_cast<int>(v));
        }
        double extent = scene_extent;
        if (!(extent > 0.0)) {
            HostCloud c = e.download();
            extent = osb::scene_extent(poses, c.positions);
        }
        osb::DeviceTrainer trainer(e, cfg, poses, planar.data(), W, H, train, test, extent);
        planar.clear();
        planar.shrink_to_fit();
        std::string metrics_path;
        // data parallel: every rank runs the loop, rank 0 alone writes osplat_train's files
        const bool writer = e.dp_rank() == 0;
        if (output_dir && writer) {
            fs::create_directories(output_dir);
            metrics_path = (fs::path(output_dir) / "metrics.jsonl").string();
            std::ofstream(metrics_path, std::ios::trunc).close();
        }
        trainer.run(start_iteration, [&](const osb::IterationReport& r) {
            // capi.cpp:207-224: metrics line + progress on log iterations, periodic checkpoints
            if (r.logged) {
                if (!metrics_path.empty()) {
                    std::ofstream out(metrics_path, std::ios::app);
                    if (!out) throw ApiError(Code::IoError, "cannot write " + metrics_path);
                    out << "{\"gaussians\":" << r.gaussians << ",\"iteration\":" << r.iteration
                        << ",\"loss\":" << json_number(r.loss) << ",\"psnr\":" << json_number(r.heldout_psnr) << "}\n";
                }
                if (progress) progress(user, r.iteration, r.loss, r.gaussians);
            }
            if (output_dir && writer && cfg.checkpoint_interval > 0 && r.iteration % cfg.checkpoint_interval == 0 &&
                r.iteration != cfg.iterations) {
                char name[64];
                std::snprintf(name, sizeof(name), "checkpoint_%06ld.ply", r.iteration);
                save_checkpoint(e.download(), (fs::path(output_dir) / name).string());
            }
        });
        if (output_dir) {
            e.dp_gather_moments();  // collective: every rank, before rank 0 writes the sidecar
            if (writer) {
                save_checkpoint(e.download(), (fs::path(output_dir) / "final.ply").string());
                osb::save_optimizer_state(e, trainer.iteration(), (fs::path(output_dir) / "final.adam").string());
            }
        }
    });
}

// osplat_eval (capi.cpp:298-306 -> run_eval, eval.cpp:63-116) over in-memory views: the split's
// views rendered one by one, each render timed with the steady clock around the call and its
// completion (the reference times render(); FPS = 1 / mean seconds), PSNR / SSIM against the
// view's image in FP64 on the device — on the panorama, or averaged over the 6 cube-face
// perspective crops of size H/2 (eval.cpp:10-19, 44-61).
osplat_status osplat_gpu_eval(osplat_gpu* ctx, size_t views, const double* transforms_cw,
                              const osplat_image* const* images, const unsigned char* is_test, const char* split,
                              int perspective_crop, osplat_report** out) {
    if (!ctx || !transforms_cw || !images || !out) return invalid("osplat_gpu_eval: null argument");
    return wrap([&] {
        const std::string sp = split ? split : "test";
        std::vector<int> idx;
        for (size_t v = 0; v < views; ++v) {
            const bool test = is_test && is_test[v];
            if (sp == "all" || (sp == "test" && test) || (sp == "train" && !test)) idx.push_back(static_cast<int>(v));
        }
        if (sp != "all" && sp != "test" && sp != "train") throw ApiError(Code::InvalidArgument, "unknown split: " + sp);
        if (idx.empty()) throw ApiError(Code::EmptySplit, "split '" + sp + "' is empty");
        Engine& e = *ctx->engine;
        osb::DeviceGuard g(e.device());
        auto rep = std::make_unique<osplat_report>();
        rep->mode = perspective_crop ? "perspective-crop" : "omnidirectional";
        const int W = images[idx[0]]->width, H = images[idx[0]]->height;
        const size_t px = static_cast<size_t>(W) * H;
        const int S = H / 2;  // cube_faces(dataset.cam.height / 2)
        const size_t crop_px = static_cast<size_t>(S) * S;
        const size_t big = std::max(px, crop_px);
        osb::DevBuf gt, crops, maps, sums;
        gt.ensure(px * 3 * sizeof(double));
        crops.ensure(crop_px * 6 * sizeof(double) + 64);
        maps.ensure(big * 15 * sizeof(double));
        sums.ensure(4 * sizeof(double));
        const double faces[6][2] = {{0.0, 0.0}, {osb::kPi / 2.0, 0.0}, {osb::kPi, 0.0}, {3.0 * osb::kPi / 2.0, 0.0},
                                    {0.0, osb::kPi / 2.0}, {0.0, -osb::kPi / 2.0}};
        auto metrics = [&](const double* a, const double* b, int w, int h, double* ps, double* ss) {
            double hs[4];
            osb::launch_metrics_f64(a, b, w, h, maps.as<double>(), sums.as<double>(), e.stream());
            OSB_CUDA_CHECK(cudaMemcpyAsync(hs, sums.as<double>(), sizeof(hs), cudaMemcpyDeviceToHost, e.stream()));
            OSB_CUDA_CHECK(cudaStreamSynchronize(e.stream()));
            const double mse = hs[0] / (static_cast<double>(w) * h * 3.0);
            *ps = mse <= 0.0 ? 99.0 : std::min(99.0, 10.0 * std::log10(1.0 / mse));
            *ss = (hs[1] / (static_cast<double>(w) * h) + hs[2] / (static_cast<double>(w) * h) +
                   hs[3] / (static_cast<double>(w) * h)) / 3.0;
        };
        double total = 0.0;
        const double bg[3] = {0.0, 0.0, 0.0};
        for (int v : idx) {
            const osplat_image* im = images[v];
            if (!im || im->width != W || im->height != H)
                throw ApiError(Code::DimensionMismatch, "evaluation images differ in size");
            double p12[12];
            checked_pose(transforms_cw + 16 * static_cast<size_t>(v), p12);
            OSB_CUDA_CHECK(cudaStreamSynchronize(e.stream()));
            const auto t0 = std::chrono::steady_clock::now();
            osb::Frame* f = e.render(p12, W, H, bg);
            try {
                e.validate(f);
                OSB_CUDA_CHECK(cudaStreamSynchronize(e.stream()));
                total += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
                OSB_CUDA_CHECK(cudaMemcpyAsync(gt.as<double>(), im->px(), px * 3 * sizeof(double),
                                               cudaMemcpyHostToDevice, e.stream()));
                const double* rgb = e.image_hwc_device(f);
                osplat_report::View rv{v, 0.0, 0.0};
                if (!perspective_crop) {
                    metrics(rgb, gt.as<double>(), W, H, &rv.psnr, &rv.ssim);
                } else {
                    double* rc = crops.as<double>();
                    double* gc = rc + crop_px * 3;
                    for (const auto& fc : faces) {
                        osb::launch_perspective_crop(rgb, W, H, S, fc[0], fc[1], rc, e.stream());
                        osb::launch_perspective_crop(gt.as<double>(), W, H, S, fc[0], fc[1], gc, e.stream());
                        double ps, ss;
                        metrics(rc, gc, S, S, &ps, &ss);
                        rv.psnr += ps;
                        rv.ssim += ss;
                    }
                    rv.psnr /= 6.0;
                    rv.ssim /= 6.0;
                }
                rep->views.push_back(rv);
                rep->mean_psnr += rv.psnr;
                rep->mean_ssim += rv.ssim;
            } catch (...) {
                e.release(f);
                throw;
            }
            e.release(f);
        }
        rep->mean_psnr /= rep->views.size();
        rep->mean_ssim /= rep->views.size();
        rep->seconds_per_frame = total / rep->views.size();
        rep->fps = rep->seconds_per_frame > 0.0 ? 1.0 / rep->seconds_per_frame : 0.0;
        *out = rep.release();
    });
}

size_t osplat_report_view_count(const osplat_report* report) { return report ? report->views.size() : 0; }

osplat_status osplat_report_view(const osplat_report* report, size_t index, int* frame_index, double* psnr,
                                 double* ssim) {
    if (!report) return invalid("osplat_report_view: null report");
    if (index >= report->views.size()) return invalid("osplat_report_view: index out of range");
    const auto& v = report->views[index];
    if (frame_index) *frame_index = v.frame_index;
    if (psnr) *psnr = v.psnr;
    if (ssim) *ssim = v.ssim;
    t_last_error.clear();
    return OSPLAT_OK;
}

osplat_status osplat_report_mean(const osplat_report* report, double* psnr, double* ssim, double* seconds_per_frame,
                                 double* fps) {
    if (!report) return invalid("osplat_report_mean: null report");
    if (psnr) *psnr = report->mean_psnr;
    if (ssim) *ssim = report->mean_ssim;
    if (seconds_per_frame) *seconds_per_frame = report->seconds_per_frame;
    if (fps) *fps = report->fps;
    t_last_error.clear();
    return OSPLAT_OK;
}

const char* osplat_report_mode(const osplat_report* report) { return report ? report->mode.c_str() : ""; }

void osplat_report_free(osplat_report* report) { delete report; }

osplat_status osplat_gpu_adam_step(osplat_gpu* ctx, const osplat_config* config, double extent, long iteration,
                                   int zero_grad) {
    if (!ctx) return invalid("osplat_gpu_adam_step: null context");
    return wrap([&] { ctx->engine->adam_step(hyper_from(config), extent, iteration, zero_grad != 0); });
}

osplat_status osplat_nccl_unique_id(unsigned char id[128]) {
    if (!id) return invalid("osplat_nccl_unique_id: null argument");
    return wrap([&] { osb::nccl_unique_id(id); });
}

osplat_status osplat_gpu_dp_init(osplat_gpu* ctx, int world, int rank, const unsigned char id[128]) {
    if (!ctx || !id) return invalid("osplat_gpu_dp_init: null argument");
    if (world < 1 || rank < 0 || rank >= world) return invalid("osplat_gpu_dp_init: rank must be in [0, world)");
    return wrap([&] { ctx->engine->dp_init(world, rank, id); });
}

osplat_status osplat_gpu_dp_step(osplat_gpu* ctx, const osplat_config* config, double extent, long iteration) {
    if (!ctx) return invalid("osplat_gpu_dp_step: null context");
    return wrap([&] { ctx->engine->dp_step(hyper_from(config), extent, iteration); });
}

osplat_status osplat_gpu_adam_step_range(osplat_gpu* ctx, const osplat_config* config, double extent, long iteration,
                                         int zero_grad, size_t begin, size_t count) {
    if (!ctx) return invalid("osplat_gpu_adam_step_range: null context");
    return wrap([&] { ctx->engine->adam_step(hyper_from(config), extent, iteration, zero_grad != 0, begin, count); });
}

osplat_status osplat_gpu_loss(osplat_gpu* ctx, const osplat_frame* frame, const float* gt, double lambda_ssim,
                              double mask, const float** d_image, double* loss) {
    if (!ctx || !frame || !gt) return invalid("osplat_gpu_loss: null argument");
    if (mask < 0.0 || mask >= 1.0) return invalid("osplat_gpu_loss: mask_bottom_fraction must be in [0, 1)");
    if (lambda_ssim < 0.0 || lambda_ssim > 1.0) return invalid("osplat_gpu_loss: lambda_ssim must be in [0, 1]");
    return wrap([&] {
        validate_frame(ctx, frame);
        Engine& e = *ctx->engine;
        double v = e.loss(frame->frame, gt, lambda_ssim, mask, loss != nullptr);
        if (loss) *loss = v;
        if (d_image) *d_image = e.d_image_buffer(static_cast<size_t>(frame->frame->W) * frame->frame->H);
    });
}

osplat_status osplat_gpu_l1_loss(osplat_gpu* ctx, const osplat_frame* frame, const float* gt, double mask,
                                 const float** d_image, double* loss) {
    return osplat_gpu_loss(ctx, frame, gt, 0.0, mask, d_image, loss);
}

namespace {
osplat_status train_view_impl(osplat_gpu* ctx, const double transform_cw[16], int width, int height, const float* gt,
                              int gt_on_device, double lambda_ssim, double mask, double* loss, double* sums_pinned);
}

osplat_status osplat_gpu_train_view(osplat_gpu* ctx, const double transform_cw[16], int width, int height,
                                    const float* gt, int gt_on_device, double lambda_ssim, double mask,
                                    double* loss) {
    return train_view_impl(ctx, transform_cw, width, height, gt, gt_on_device, lambda_ssim, mask, loss, nullptr);
}

osplat_status osplat_gpu_train_view_async(osplat_gpu* ctx, const double transform_cw[16], int width, int height,
                                          const float* gt, int gt_on_device, double lambda_ssim, double mask,
                                          double* loss_sums) {
    return train_view_impl(ctx, transform_cw, width, height, gt, gt_on_device, lambda_ssim, mask, nullptr,
                           loss_sums ? loss_sums : nullptr);
}

double osplat_loss_value(const double sums[4], double lambda_ssim, int width, int height, double mask) {
    // trainer.cpp:54-63, as Engine::loss_value
    const int masked = static_cast<int>(std::floor(mask * height));
    const double npx = static_cast<double>(width) * (height - masked);
    const double n = npx * 3.0;
    double value = (1.0 - lambda_ssim) * (sums[0] / n);
    if (lambda_ssim > 0.0) value += lambda_ssim * (1.0 - ((sums[1] + sums[2] + sums[3]) / npx) / 3.0);
    return value;
}

namespace {
osplat_status train_view_impl(osplat_gpu* ctx, const double transform_cw[16], int width, int height, const float* gt,
                              int gt_on_device, double lambda_ssim, double mask, double* loss, double* sums_pinned) {
    if (!ctx || !transform_cw || !gt) return invalid("osplat_gpu_train_view: null argument");
    if (lambda_ssim < 0.0 || lambda_ssim > 1.0) return invalid("osplat_gpu_train_view: lambda_ssim must be in [0, 1]");
    if (mask < 0.0 || mask >= 1.0) return invalid("osplat_gpu_train_view: mask_bottom_fraction must be in [0, 1)");
    return wrap([&] {
        check_dims(width, height);
        double p12[12];
        checked_pose(transform_cw, p12);
        Engine& e = *ctx->engine;
        osb::DeviceGuard g(e.device());
        const size_t plane = static_cast<size_t>(width) * height;
        // a host target is uploaded on the copy stream while K1-K3 run (overlapped H2D)
        const float* gt_dev = gt_on_device ? gt : e.upload_target_async(gt, plane);
        const double zero[3] = {0, 0, 0};
        osb::Frame* f = e.render(p12, width, height, zero);
        try {
            if (!gt_on_device) e.wait_target();
            const double v = e.loss(f, gt_dev, lambda_ssim, mask, false);
            (void)v;
            if (!gt_on_device) e.release_target();
            const size_t pixels = plane;
            e.backward(f, e.d_image_buffer(pixels), true);
            if (loss) {
                // the L1 sum lives on the device; one 8-byte read completes the step
                *loss = e.loss_value(f, mask);
            }
            if (sums_pinned) e.loss_sums_async(sums_pinned);  // no wait: read after osplat_gpu_synchronize
        } catch (...) {
            e.release(f);
            throw;
        }
        e.release(f);
    });
}
}  // namespace

osplat_status osplat_gpu_profile(osplat_gpu* ctx, int timing, int count_work) {
    if (!ctx) return invalid("osplat_gpu_profile: null context");
    return wrap([&] { ctx->engine->set_profiling(timing != 0, count_work != 0); });
}

osplat_status osplat_gpu_profile_read(osplat_gpu* ctx, double* ms, long* launches, int reset) {
    if (!ctx) return invalid("osplat_gpu_profile_read: null context");
    return wrap([&] { ctx->engine->profile_read(ms, launches, reset != 0); });
}

const char* osplat_kernel_name(int id) { return osb::kernel_name(id); }

osplat_status osplat_frame_work(const osplat_frame* frame, uint64_t* fwd, uint64_t* bwd, uint64_t* instances) {
    if (!frame) return invalid("osplat_frame_work: null frame");
    return wrap([&] {
        frame->engine->validate(frame->frame);
        const osb::Frame& f = *frame->frame;
        if (!f.count_work) throw ApiError(Code::StateMismatch, "frame was rendered without work counting");
        osb::DeviceGuard g(frame->engine->device());
        cudaStream_t s = frame->engine->stream();
        unsigned long long host[2] = {0, 0};
        osb::launch_work_count(f.fb(), f.W * f.H, f.work.as<unsigned long long>(), s);
        OSB_CUDA_CHECK(cudaMemcpyAsync(host, f.work.as<void>(), 16, cudaMemcpyDeviceToHost, s));
        OSB_CUDA_CHECK(cudaStreamSynchronize(s));
        if (fwd) *fwd = host[0];
        if (bwd) *bwd = host[1];
        if (instances) *instances = f.M;
    });
}

long long osplat_gpu_launch_count(void) { return osb::launches_total(); }

}  // extern "C"
