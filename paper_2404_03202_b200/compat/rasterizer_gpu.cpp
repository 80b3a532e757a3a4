// rasterizer_gpu.cpp — the reference's C++ rasterizer API (proj/include/omnisplat/rasterizer.hpp:72-94)
// served by this library: project_gaussian, bin_to_tiles, blend_forward and render run on the
// B200 through the C ABI (include/osplat.h). Compiled against the reference's own headers, it
// replaces proj/src/rasterizer.cpp in a build of the reference, so code written
// against omnisplat::render — the reference's tests, trainer, eval — runs on the GPU unchanged.
//
// Contract differences: Gaussian parameters are stored as FP32 on the device (the
// projection geometry is FP64 from those values), colour and transmittance come back as the FP32
// values the blend produced, and tile_size must be 16 (UnsupportedFormat otherwise). reference_render
// (the brute-force oracle) is not part of this file.
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <optional>
#include <string>
#include <vector>

#include "omnisplat/error.hpp"
#include "omnisplat/rasterizer.hpp"
#include "osplat.h"

namespace omnisplat {
namespace {

// osplat_status + "<ErrorCode>: message" (capi.cpp:41-66 mapping) back to the reference's Error.
void check(osplat_status st) {
    if (st == OSPLAT_OK) return;
    const std::string msg = osplat_last_error() ? osplat_last_error() : "";
    for (int c = 0; c <= static_cast<int>(ErrorCode::InvalidArgument); ++c) {
        const std::string name = error_code_name(static_cast<ErrorCode>(c));
        if (msg.compare(0, name.size() + 2, name + ": ") == 0) throw Error(static_cast<ErrorCode>(c), msg);
    }
    switch (st) {
        case OSPLAT_ERR_INVALID_ARGUMENT: throw Error(ErrorCode::InvalidArgument, msg);
        case OSPLAT_ERR_IO: throw Error(ErrorCode::IoError, msg);
        case OSPLAT_ERR_PARSE: throw Error(ErrorCode::ParseError, msg);
        case OSPLAT_ERR_VALIDATION: throw Error(ErrorCode::ValidationError, msg);
        case OSPLAT_ERR_UNSUPPORTED: throw Error(ErrorCode::UnsupportedFormat, msg);
        default: throw std::runtime_error(msg);
    }
}

// One device context for the process (device OSPLAT_DEVICE, default 0), created on first use.
// The reference's calls are not concurrent on one cloud; the mutex keeps two host
// threads from interleaving uploads and renders on the shared context.
struct Device {
    std::mutex mu;
    osplat_gpu* ctx = nullptr;
    Device() {
        const char* env = std::getenv("OSPLAT_DEVICE");
        osplat_cloud* empty = nullptr;
        check(osplat_cloud_create(0, 0, 0, nullptr, nullptr, nullptr, nullptr, nullptr, &empty));
        const osplat_status st = osplat_gpu_create(env ? std::atoi(env) : 0, nullptr, empty, &ctx);
        osplat_cloud_free(empty);
        check(st);
    }
    ~Device() { osplat_gpu_free(ctx); }
};

Device& device() {
    static Device d;
    return d;
}

struct Frame {
    osplat_frame* f = nullptr;
    ~Frame() { osplat_frame_free(f); }
};

void require_tile16(int tile_size) {
    if (tile_size != kDefaultTileSize || kDefaultTileSize != 16)
        throw Error(ErrorCode::UnsupportedFormat, "UnsupportedFormat: tile_size must be 16 on the GPU path");
}

// GaussianCloud (scene.hpp:31-55) -> the device context, Gaussians [first, first + count).
void upload(osplat_gpu* ctx, const GaussianCloud& cloud, size_t first, size_t count) {
    const size_t bc = static_cast<size_t>(cloud.basis_count());
    std::vector<double> pos(3 * count), sh(3 * bc * count), rot(4 * count), ls(3 * count), op(count);
    for (size_t k = 0; k < count; ++k) {
        const size_t i = first + k;
        const Vec3& m = cloud.positions[i];
        pos[3 * k] = m.x, pos[3 * k + 1] = m.y, pos[3 * k + 2] = m.z;
        for (size_t b = 0; b < bc; ++b) {
            const Vec3& c = cloud.sh_coeffs[i * bc + b];
            sh[(k * bc + b) * 3] = c.x, sh[(k * bc + b) * 3 + 1] = c.y, sh[(k * bc + b) * 3 + 2] = c.z;
        }
        const Vec4& q = cloud.rotations[i];
        rot[4 * k] = q.w, rot[4 * k + 1] = q.x, rot[4 * k + 2] = q.y, rot[4 * k + 3] = q.z;
        const Vec3& l = cloud.log_scales[i];
        ls[3 * k] = l.x, ls[3 * k + 1] = l.y, ls[3 * k + 2] = l.z;
        op[k] = cloud.opacity_logits[i];
    }
    osplat_cloud* c = nullptr;
    check(osplat_cloud_create(count, cloud.sh_degree, cloud.active_sh_degree, pos.data(), sh.data(), rot.data(),
                              ls.data(), op.data(), &c));
    const osplat_status st = osplat_gpu_upload(ctx, c);
    osplat_cloud_free(c);
    check(st);
}

void transform_of(const Pose& pose, double T[16]) {
    for (int r = 0; r < 3; ++r) {
        for (int c = 0; c < 3; ++c) T[4 * r + c] = pose.rotation.m[3 * r + c];
    }
    T[3] = pose.translation.x, T[7] = pose.translation.y, T[11] = pose.translation.z;
    T[12] = T[13] = T[14] = 0.0;
    T[15] = 1.0;
}

// SplatProjection records of a frame (osplat_frame_splats), in the frame's record order.
std::vector<SplatProjection> splats_of(osplat_frame* f) {
    size_t n = 0;
    check(osplat_frame_splats(f, &n, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr));
    std::vector<int32_t> id(n);
    std::vector<double> p(2 * n), cov(3 * n), conic(3 * n), radius(n), depth(n), color(3 * n), alpha(n), t(3 * n);
    check(osplat_frame_splats(f, &n, id.data(), p.data(), cov.data(), conic.data(), radius.data(), depth.data(),
                              color.data(), alpha.data(), t.data()));
    std::vector<SplatProjection> out(n);
    for (size_t i = 0; i < n; ++i) {
        SplatProjection& s = out[i];
        s.gaussian_id = id[i];
        s.p = {p[2 * i], p[2 * i + 1]};
        s.cov = {cov[3 * i], cov[3 * i + 1], cov[3 * i + 2]};
        s.conic = {conic[3 * i], conic[3 * i + 1], conic[3 * i + 2]};
        s.radius = radius[i];
        s.depth = depth[i];
        s.color = {color[3 * i], color[3 * i + 1], color[3 * i + 2]};
        s.alpha_base = alpha[i];
        s.t = {t[3 * i], t[3 * i + 1], t[3 * i + 2]};
    }
    return out;
}

// The frame's sorted tile lists as a TileGrid; `remap` turns device ids into projection indices.
TileGrid grid_of(osplat_frame* f, const std::vector<int>* remap) {
    TileGrid g;
    g.tile_size = 16;
    size_t M = 0;
    check(osplat_frame_tiles(f, &g.tiles_x, &g.tiles_y, &M, nullptr, nullptr));
    std::vector<uint32_t> ranges(2 * static_cast<size_t>(g.tile_count())), ids(M);
    check(osplat_frame_tiles(f, nullptr, nullptr, &M, ranges.data(), ids.data()));
    g.tiles.assign(static_cast<size_t>(g.tile_count()), {});
    for (size_t t = 0; t < g.tiles.size(); ++t) {
        auto& list = g.tiles[t];
        for (uint32_t e = ranges[2 * t]; e < ranges[2 * t + 1]; ++e)
            list.push_back(remap ? (*remap)[ids[e]] : static_cast<int>(ids[e]));
    }
    return g;
}

void pixels_of(osplat_frame* f, const EquirectCamera& cam, RenderOutput& out) {
    const size_t px = static_cast<size_t>(cam.width) * cam.height;
    out.color = Image(cam.width, cam.height);
    check(osplat_frame_image(f, out.color.data.data()));
    std::vector<float> T(px);
    out.contributors.assign(px, 0);
    out.last_contrib.assign(px, 0);
    check(osplat_frame_pixels(f, nullptr, T.data(), out.contributors.data(), out.last_contrib.data()));
    out.transmittance.assign(T.begin(), T.end());
}

Frame render_projections(osplat_gpu* ctx, const std::vector<SplatProjection>& prs, const EquirectCamera& cam,
                         const Vec3& bg, const TileGrid* grid) {
    const size_t n = prs.size();
    std::vector<int32_t> id(n);
    std::vector<double> p(2 * n), cov(3 * n), conic(3 * n), radius(n), depth(n), color(3 * n), alpha(n);
    for (size_t i = 0; i < n; ++i) {
        const SplatProjection& s = prs[i];
        id[i] = s.gaussian_id;
        p[2 * i] = s.p.x, p[2 * i + 1] = s.p.y;
        cov[3 * i] = s.cov.a, cov[3 * i + 1] = s.cov.b, cov[3 * i + 2] = s.cov.c;
        conic[3 * i] = s.conic.a, conic[3 * i + 1] = s.conic.b, conic[3 * i + 2] = s.conic.c;
        radius[i] = s.radius;
        depth[i] = s.depth;
        color[3 * i] = s.color.x, color[3 * i + 1] = s.color.y, color[3 * i + 2] = s.color.z;
        alpha[i] = s.alpha_base;
    }
    std::vector<uint32_t> offsets;
    std::vector<int32_t> entries;
    if (grid) {
        require_tile16(grid->tile_size);
        if (grid->tiles_x != (cam.width + 15) / 16 || grid->tiles_y != (cam.height + 15) / 16 ||
            grid->tiles.size() != static_cast<size_t>(grid->tile_count()))
            throw Error(ErrorCode::DimensionMismatch, "DimensionMismatch: tile grid does not match the camera");
        offsets.push_back(0);
        for (const auto& list : grid->tiles) {
            entries.insert(entries.end(), list.begin(), list.end());
            offsets.push_back(static_cast<uint32_t>(entries.size()));
        }
    }
    const double background[3] = {bg.x, bg.y, bg.z};
    Frame fr;
    check(osplat_gpu_render_projected(ctx, n, id.data(), p.data(), cov.data(), conic.data(), radius.data(),
                                      depth.data(), color.data(), alpha.data(), cam.width, cam.height, background,
                                      grid ? offsets.data() : nullptr, grid ? entries.data() : nullptr, &fr.f));
    return fr;
}

}  // namespace

std::optional<SplatProjection> project_gaussian(const GaussianCloud& cloud, std::size_t index, const Pose& pose,
                                                const EquirectCamera& cam) {
    if (index >= cloud.size()) throw Error(ErrorCode::OutOfBounds, "OutOfBounds: Gaussian index");
    Device& d = device();
    std::lock_guard<std::mutex> lock(d.mu);
    upload(d.ctx, cloud, index, 1);
    double T[16];
    transform_of(pose, T);
    Frame fr;
    check(osplat_gpu_render(d.ctx, T, cam.width, cam.height, nullptr, &fr.f));
    std::vector<SplatProjection> s = splats_of(fr.f);
    if (s.empty()) return std::nullopt;
    s[0].gaussian_id = static_cast<int>(index);
    return s[0];
}

TileGrid bin_to_tiles(const std::vector<SplatProjection>& projections, const EquirectCamera& cam, int tile_size) {
    require_tile16(tile_size);
    Device& d = device();
    std::lock_guard<std::mutex> lock(d.mu);
    Frame fr = render_projections(d.ctx, projections, cam, Vec3{0, 0, 0}, nullptr);
    return grid_of(fr.f, nullptr);  // ids of a projection frame are already record indices
}

RenderOutput blend_forward(TileGrid grid, std::vector<SplatProjection> projections, const EquirectCamera& cam,
                           const RenderSettings& settings) {
    require_tile16(settings.tile_size);
    Device& d = device();
    std::lock_guard<std::mutex> lock(d.mu);
    RenderOutput out;
    {
        Frame fr = render_projections(d.ctx, projections, cam, settings.background, &grid);
        pixels_of(fr.f, cam, out);
    }
    out.camera = cam;
    out.background = settings.background;
    out.grid = std::move(grid);
    out.projections = std::move(projections);
    return out;
}

RenderOutput render(const GaussianCloud& cloud, const Pose& pose, const EquirectCamera& cam,
                    const RenderSettings& settings) {
    require_tile16(settings.tile_size);
    Device& d = device();
    std::lock_guard<std::mutex> lock(d.mu);
    upload(d.ctx, cloud, 0, cloud.size());
    double T[16];
    transform_of(pose, T);
    const double bg[3] = {settings.background.x, settings.background.y, settings.background.z};
    Frame fr;
    check(osplat_gpu_render(d.ctx, T, cam.width, cam.height, bg, &fr.f));
    RenderOutput out;
    pixels_of(fr.f, cam, out);
    out.projections = splats_of(fr.f);
    // tile lists hold Gaussian ids on the device; the reference's hold projection indices
    std::vector<int> index_of(cloud.size(), -1);
    for (size_t k = 0; k < out.projections.size(); ++k) index_of[out.projections[k].gaussian_id] = static_cast<int>(k);
    out.grid = grid_of(fr.f, &index_of);
    out.cloud_size = cloud.size();
    out.pose = pose;
    out.camera = cam;
    out.background = settings.background;
    return out;
}

}  // namespace omnisplat
