// ref_shim.cpp — TEST INFRASTRUCTURE ONLY. Exposes the reference's own C++ hot path
// (render / reference_render / backward / adam_step / loss from /root/reference/proj/src)
// through oracle/oracle.h so tests can diff the C restatement and the CUDA product against
// the unmodified reference code. Built by oracle/Makefile into oracle/_ref/libref_oracle.so;
// the reference sources are compiled where they lie and never copied into this repo.
#include <chrono>
#include <cstring>
#include <random>
#include <vector>

#include "omnisplat/dataio.hpp"
#include "omnisplat/eval.hpp"
#include "omnisplat/gradients.hpp"
#include "omnisplat/metrics.hpp"
#include "omnisplat/parallel.hpp"
#include "omnisplat/rasterizer.hpp"
#include "omnisplat/trainer.hpp"

#include "oracle.h"

using namespace omnisplat;

struct oracle_frame {
    RenderOutput out;
};

namespace {

GaussianCloud to_cloud(const oracle_cloud* c) {
    GaussianCloud g;
    g.sh_degree = c->sh_degree;
    g.active_sh_degree = c->active_sh_degree;
    g.resize(static_cast<std::size_t>(c->n));
    const int bc = g.basis_count();
    for (int i = 0; i < c->n; ++i) {
        g.positions[i] = {c->positions[3 * i], c->positions[3 * i + 1], c->positions[3 * i + 2]};
        g.rotations[i] = {c->rotations[4 * i], c->rotations[4 * i + 1], c->rotations[4 * i + 2],
                          c->rotations[4 * i + 3]};
        g.log_scales[i] = {c->log_scales[3 * i], c->log_scales[3 * i + 1], c->log_scales[3 * i + 2]};
        g.opacity_logits[i] = c->opacity_logits[i];
        for (int b = 0; b < bc; ++b) {
            const double* s = c->sh + (static_cast<std::size_t>(i) * bc + b) * 3;
            g.sh_coeffs[static_cast<std::size_t>(i) * bc + b] = {s[0], s[1], s[2]};
        }
    }
    return g;
}

void from_cloud(const GaussianCloud& g, oracle_cloud* c) {
    const int bc = g.basis_count();
    for (std::size_t i = 0; i < g.size(); ++i) {
        for (int k = 0; k < 3; ++k) c->positions[3 * i + k] = g.positions[i][k];
        for (int k = 0; k < 4; ++k) c->rotations[4 * i + k] = g.rotations[i][k];
        for (int k = 0; k < 3; ++k) c->log_scales[3 * i + k] = g.log_scales[i][k];
        c->opacity_logits[i] = g.opacity_logits[i];
        for (int b = 0; b < bc; ++b)
            for (int k = 0; k < 3; ++k) c->sh[(i * bc + b) * 3 + k] = g.sh_coeffs[i * bc + b][k];
    }
}

double g_last_seconds = 0.0;

struct Stopwatch {
    std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
    ~Stopwatch() {
        g_last_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    }
};

Pose to_pose(const double* p) {
    Pose pose;
    for (int i = 0; i < 9; ++i) pose.rotation.m[i] = p[i];
    pose.translation = {p[9], p[10], p[11]};
    return pose;
}

}  // namespace

extern "C" {

oracle_frame* oracle_render(const oracle_cloud* c, const double pose[12], int w, int h, const double bg[3]) {
    try {
        RenderSettings s;
        if (bg) s.background = {bg[0], bg[1], bg[2]};
        auto* f = new oracle_frame;
        GaussianCloud cloud = to_cloud(c);
        Pose p = to_pose(pose);
        {
            Stopwatch sw;
            f->out = render(cloud, p, EquirectCamera{w, h}, s);
        }
        return f;
    } catch (...) {
        return nullptr;
    }
}

oracle_frame* oracle_blend_projections(int n, const int* gid, const double* p, const double* cov,
                                       const double* conic, const double* radius, const double* depth,
                                       const double* color, const double* alpha, int w, int h, const double bg[3],
                                       const long* offsets, const int* items) {
    try {
        std::vector<SplatProjection> prs(static_cast<size_t>(n));
        for (int i = 0; i < n; ++i) {
            SplatProjection& s = prs[i];
            s.gaussian_id = gid ? gid[i] : i;
            s.p = {p[2 * i], p[2 * i + 1]};
            s.cov = {cov[3 * i], cov[3 * i + 1], cov[3 * i + 2]};
            s.conic = {conic[3 * i], conic[3 * i + 1], conic[3 * i + 2]};
            s.radius = radius[i];
            s.depth = depth[i];
            s.color = {color[3 * i], color[3 * i + 1], color[3 * i + 2]};
            s.alpha_base = alpha[i];
        }
        EquirectCamera cam{w, h};
        RenderSettings st;
        if (bg) st.background = {bg[0], bg[1], bg[2]};
        TileGrid grid;
        if (offsets) {
            grid.tile_size = 16;
            grid.tiles_x = (w + 15) / 16;
            grid.tiles_y = (h + 15) / 16;
            grid.tiles.resize(static_cast<size_t>(grid.tile_count()));
            for (int t = 0; t < grid.tile_count(); ++t) grid.tiles[t].assign(items + offsets[t], items + offsets[t + 1]);
        } else {
            grid = bin_to_tiles(prs, cam, 16);
        }
        auto* f = new oracle_frame;
        f->out = blend_forward(std::move(grid), std::move(prs), cam, st);
        return f;
    } catch (...) {
        return nullptr;
    }
}

oracle_frame* oracle_reference_render(const oracle_cloud* c, const double pose[12], int w, int h,
                                      const double bg[3]) {
    try {
        RenderSettings s;
        if (bg) s.background = {bg[0], bg[1], bg[2]};
        auto* f = new oracle_frame;
        f->out = reference_render(to_cloud(c), to_pose(pose), EquirectCamera{w, h}, s);
        return f;
    } catch (...) {
        return nullptr;
    }
}

void oracle_frame_free(oracle_frame* f) { delete f; }

int oracle_frame_num_projections(const oracle_frame* f) {
    return f ? static_cast<int>(f->out.projections.size()) : 0;
}

void oracle_frame_projections(const oracle_frame* f, int* gid, double* p, double* cov, double* conic,
                              double* radius, double* depth, double* color, double* alpha, double* t) {
    const auto& pr = f->out.projections;
    for (std::size_t i = 0; i < pr.size(); ++i) {
        const SplatProjection& s = pr[i];
        if (gid) gid[i] = s.gaussian_id;
        if (p) { p[2 * i] = s.p.x; p[2 * i + 1] = s.p.y; }
        if (cov) { cov[3 * i] = s.cov.a; cov[3 * i + 1] = s.cov.b; cov[3 * i + 2] = s.cov.c; }
        if (conic) { conic[3 * i] = s.conic.a; conic[3 * i + 1] = s.conic.b; conic[3 * i + 2] = s.conic.c; }
        if (radius) radius[i] = s.radius;
        if (depth) depth[i] = s.depth;
        if (color) for (int k = 0; k < 3; ++k) color[3 * i + k] = s.color[k];
        if (alpha) alpha[i] = s.alpha_base;
        if (t) for (int k = 0; k < 3; ++k) t[3 * i + k] = s.t[k];
    }
}

long oracle_frame_tile_count(const oracle_frame* f, int* tx, int* ty) {
    if (tx) *tx = f->out.grid.tiles_x;
    if (ty) *ty = f->out.grid.tiles_y;
    long m = 0;
    for (const auto& t : f->out.grid.tiles) m += static_cast<long>(t.size());
    return m;
}

void oracle_frame_tile_lists(const oracle_frame* f, long* offsets, int* items) {
    long o = 0;
    std::size_t ti = 0;
    for (const auto& t : f->out.grid.tiles) {
        if (offsets) offsets[ti] = o;
        for (int v : t) {
            if (items) items[o] = v;
            ++o;
        }
        ++ti;
    }
    if (offsets) offsets[ti] = o;
}

void oracle_frame_pixels(const oracle_frame* f, double* rgb, double* T, int* contrib, int* last) {
    const RenderOutput& r = f->out;
    std::size_t px = r.color.pixel_count();
    if (rgb) std::memcpy(rgb, r.color.data.data(), px * 3 * sizeof(double));
    if (T) std::memcpy(T, r.transmittance.data(), px * sizeof(double));
    if (contrib) std::memcpy(contrib, r.contributors.data(), px * sizeof(int));
    if (last) {
        if (r.last_contrib.size() == px)
            std::memcpy(last, r.last_contrib.data(), px * sizeof(int));
        else
            std::memset(last, 0, px * sizeof(int));
    }
}

int oracle_backward(const oracle_frame* f, const double* d_image, const oracle_cloud* c,
                    const double pose[12], int w, int h, oracle_grads* g) {
    try {
        GaussianCloud cloud = to_cloud(c);
        Image di(w, h);
        std::memcpy(di.data.data(), d_image, di.data.size() * sizeof(double));
        GradientBuffer buf;
        buf.resize(cloud.size(), cloud.basis_count());
        for (int i = 0; i < c->n; ++i) {
            buf.screen_norm_sum[i] = g->screen_norm_sum[i];
            buf.screen_hits[i] = g->screen_hits[i];
        }
        {
            Stopwatch sw;
            backward(f->out, di, cloud, to_pose(pose), EquirectCamera{w, h}, buf);
        }
        const int bc = cloud.basis_count();
        for (int i = 0; i < c->n; ++i) {
            for (int k = 0; k < 3; ++k) g->d_position[3 * i + k] = buf.d_position[i][k];
            for (int k = 0; k < 4; ++k) g->d_rotation[4 * i + k] = buf.d_rotation[i][k];
            for (int k = 0; k < 3; ++k) g->d_log_scale[3 * i + k] = buf.d_log_scale[i][k];
            g->d_opacity_logit[i] = buf.d_opacity_logit[i];
            g->d_screen[2 * i] = buf.d_screen[i].x;
            g->d_screen[2 * i + 1] = buf.d_screen[i].y;
            g->screen_norm_sum[i] = buf.screen_norm_sum[i];
            g->screen_hits[i] = buf.screen_hits[i];
            for (int b = 0; b < bc; ++b)
                for (int k = 0; k < 3; ++k)
                    g->d_sh[(static_cast<std::size_t>(i) * bc + b) * 3 + k] =
                        buf.d_sh[static_cast<std::size_t>(i) * bc + b][k];
        }
        return 0;
    } catch (...) {
        return 1;
    }
}

void oracle_adam_step(oracle_cloud* c, const oracle_grads* g, oracle_adam* st, const oracle_adam_cfg* cfg,
                      double extent, long iteration) {
    GaussianCloud cloud = to_cloud(c);
    const int bc = cloud.basis_count();
    const std::size_t n = cloud.size();
    GradientBuffer buf;
    buf.resize(n, bc);
    for (std::size_t i = 0; i < n; ++i) {
        buf.d_position[i] = {g->d_position[3 * i], g->d_position[3 * i + 1], g->d_position[3 * i + 2]};
        buf.d_rotation[i] = {g->d_rotation[4 * i], g->d_rotation[4 * i + 1], g->d_rotation[4 * i + 2],
                             g->d_rotation[4 * i + 3]};
        buf.d_log_scale[i] = {g->d_log_scale[3 * i], g->d_log_scale[3 * i + 1], g->d_log_scale[3 * i + 2]};
        buf.d_opacity_logit[i] = g->d_opacity_logit[i];
        for (int b = 0; b < bc; ++b) {
            const double* s = g->d_sh + (i * bc + b) * 3;
            buf.d_sh[i * bc + b] = {s[0], s[1], s[2]};
        }
    }
    AdamState state;
    state.step = st->step;
    auto load = [&](std::vector<double>& v, const double* src, std::size_t k) { v.assign(src, src + k); };
    load(state.m_position, st->m_position, n * 3);
    load(state.v_position, st->v_position, n * 3);
    load(state.m_sh, st->m_sh, n * 3 * bc);
    load(state.v_sh, st->v_sh, n * 3 * bc);
    load(state.m_rotation, st->m_rotation, n * 4);
    load(state.v_rotation, st->v_rotation, n * 4);
    load(state.m_scale, st->m_scale, n * 3);
    load(state.v_scale, st->v_scale, n * 3);
    load(state.m_opacity, st->m_opacity, n);
    load(state.v_opacity, st->v_opacity, n);
    TrainConfig tc;
    tc.iterations = cfg->iterations;
    tc.lr_position_init = cfg->lr_position_init;
    tc.lr_position_final = cfg->lr_position_final;
    tc.lr_sh_dc = cfg->lr_sh_dc;
    tc.lr_sh_rest = cfg->lr_sh_rest;
    tc.lr_opacity = cfg->lr_opacity;
    tc.lr_scale = cfg->lr_scale;
    tc.lr_rotation = cfg->lr_rotation;
    {
        Stopwatch sw;
        adam_step(cloud, buf, state, tc, extent, iteration);
    }
    from_cloud(cloud, c);
    st->step = state.step;
    auto store = [](const std::vector<double>& v, double* dst) { std::memcpy(dst, v.data(), v.size() * 8); };
    store(state.m_position, st->m_position);
    store(state.v_position, st->v_position);
    store(state.m_sh, st->m_sh);
    store(state.v_sh, st->v_sh);
    store(state.m_rotation, st->m_rotation);
    store(state.v_rotation, st->v_rotation);
    store(state.m_scale, st->m_scale);
    store(state.v_scale, st->v_scale);
    store(state.m_opacity, st->m_opacity);
    store(state.v_opacity, st->v_opacity);
}

double oracle_loss(const double* r, const double* gt, int w, int h, double lambda, double mask,
                   double* d_image) {
    Image a(w, h), b(w, h);
    std::memcpy(a.data.data(), r, a.data.size() * 8);
    std::memcpy(b.data.data(), gt, b.data.size() * 8);
    LossResult lr;
    {
        Stopwatch sw;
        lr = loss(a, b, lambda, mask);
    }
    if (d_image) std::memcpy(d_image, lr.d_image.data.data(), lr.d_image.data.size() * 8);
    return lr.value;
}

// cube_faces(size) + perspective_crop (eval.cpp:10-61): the 6 S x S x 3 crops of an H x W x 3 panorama.
void oracle_ref_cube_crops(const double* pano, int w, int h, int size, double* out) {
    Image p(w, h);
    std::memcpy(p.data.data(), pano, p.data.size() * 8);
    const auto faces = cube_faces(size);
    for (std::size_t k = 0; k < faces.size(); ++k) {
        Image c = perspective_crop(p, faces[k]);
        std::memcpy(out + k * c.data.size(), c.data.data(), c.data.size() * 8);
    }
}

void oracle_metrics(const double* a, const double* b, int w, int h, double* out_psnr, double* out_ssim) {
    Image x(w, h), y(w, h);
    std::memcpy(x.data.data(), a, x.data.size() * 8);
    std::memcpy(y.data.data(), b, y.data.size() * 8);
    if (out_psnr) *out_psnr = psnr(x, y);
    if (out_ssim) *out_ssim = ssim(x, y);
}

int oracle_densify_and_prune(const oracle_cloud* in, const double* norm_sum, const long* hits,
                             const double* max_radius, const oracle_adam* st, const oracle_densify_cfg* cfg,
                             double extent, unsigned long long seed, int radius_active, oracle_cloud* out,
                             oracle_adam* st_out, oracle_edit* summary) {
    GaussianCloud cloud = to_cloud(in);
    const int bc = cloud.basis_count();
    const std::size_t n = cloud.size();
    GradientBuffer buf;
    buf.resize(n, bc);
    for (std::size_t i = 0; i < n; ++i) {
        buf.screen_norm_sum[i] = norm_sum[i];
        buf.screen_hits[i] = hits[i];
    }
    DensifyStats stats;
    stats.resize(n);
    for (std::size_t i = 0; i < n; ++i) stats.max_radius_px[i] = max_radius[i];
    AdamState state;
    state.step = st->step;
    auto load = [&](std::vector<double>& v, const double* src, std::size_t k) { v.assign(src, src + k); };
    load(state.m_position, st->m_position, n * 3);
    load(state.v_position, st->v_position, n * 3);
    load(state.m_sh, st->m_sh, n * 3 * bc);
    load(state.v_sh, st->v_sh, n * 3 * bc);
    load(state.m_rotation, st->m_rotation, n * 4);
    load(state.v_rotation, st->v_rotation, n * 4);
    load(state.m_scale, st->m_scale, n * 3);
    load(state.v_scale, st->v_scale, n * 3);
    load(state.m_opacity, st->m_opacity, n);
    load(state.v_opacity, st->v_opacity, n);
    TrainConfig tc;
    tc.densify_grad_threshold = cfg->densify_grad_threshold;
    tc.scale_split_threshold = cfg->scale_split_threshold;
    tc.split_factor = cfg->split_factor;
    tc.prune_opacity = cfg->prune_opacity;
    tc.prune_scale_world = cfg->prune_scale_world;
    tc.prune_radius_px = cfg->prune_radius_px;
    std::mt19937_64 rng(seed);
    EditSummary e;
    {
        Stopwatch sw;
        e = densify_and_prune(cloud, buf, stats, state, tc, extent, rng, radius_active != 0);
    }
    out->n = static_cast<int>(cloud.size());
    out->sh_degree = cloud.sh_degree;
    out->active_sh_degree = cloud.active_sh_degree;
    from_cloud(cloud, out);
    st_out->step = state.step;
    auto store = [](const std::vector<double>& v, double* dst) { std::memcpy(dst, v.data(), v.size() * 8); };
    store(state.m_position, st_out->m_position);
    store(state.v_position, st_out->v_position);
    store(state.m_sh, st_out->m_sh);
    store(state.v_sh, st_out->v_sh);
    store(state.m_rotation, st_out->m_rotation);
    store(state.v_rotation, st_out->v_rotation);
    store(state.m_scale, st_out->m_scale);
    store(state.v_scale, st_out->v_scale);
    store(state.m_opacity, st_out->m_opacity);
    store(state.v_opacity, st_out->v_opacity);
    summary->cloned = e.cloned;
    summary->split = e.split;
    summary->pruned = e.pruned;
    summary->final_count = static_cast<long>(e.final_count);
    return 0;
}

void oracle_reset_opacity(oracle_cloud* c, double ceiling) {
    GaussianCloud cloud = to_cloud(c);
    reset_opacity(cloud, ceiling);
    from_cloud(cloud, c);
}

int oracle_ref_save_checkpoint(const oracle_cloud* c, const char* path) {
    try {
        save_checkpoint(to_cloud(c), path);
        return 0;
    } catch (...) {
        return 1;
    }
}

int oracle_ref_save_optimizer_state(const oracle_adam* st, int n, int bc, long iteration, const char* path) {
    AdamState s;
    s.step = st->step;
    const std::size_t N = static_cast<std::size_t>(n);
    auto load = [&](std::vector<double>& v, const double* src, std::size_t k) { v.assign(src, src + k); };
    load(s.m_position, st->m_position, N * 3);
    load(s.v_position, st->v_position, N * 3);
    load(s.m_sh, st->m_sh, N * 3 * bc);
    load(s.v_sh, st->v_sh, N * 3 * bc);
    load(s.m_rotation, st->m_rotation, N * 4);
    load(s.v_rotation, st->v_rotation, N * 4);
    load(s.m_scale, st->m_scale, N * 3);
    load(s.v_scale, st->v_scale, N * 3);
    load(s.m_opacity, st->m_opacity, N);
    load(s.v_opacity, st->v_opacity, N);
    try {
        save_optimizer_state(s, iteration, bc, path);
        return 0;
    } catch (...) {
        return 1;
    }
}

void oracle_mt64_draws(unsigned long long seed, long count, unsigned long long* out) {
    std::mt19937_64 rng(seed);
    for (long i = 0; i < count; ++i) out[i] = rng();
}

unsigned long long oracle_mix64(unsigned long long x) {
    // trainer.cpp:300-306 lives in an anonymous namespace there; restated for the RNG seeds
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

void oracle_set_threads(int n) { set_thread_count(n); }
double oracle_last_seconds(void) { return g_last_seconds; }
int oracle_threads(void) { return thread_count(); }
const char* oracle_kind(void) { return "reference"; }

}  // extern "C"
