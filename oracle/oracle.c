/* oracle.c — TEST INFRASTRUCTURE ONLY: a plain-C, FP64, single-threaded restatement of the
 * reference ERP splatting path, used as the parity checker for the CUDA product.
 * It is never linked into the product library.
 *
 * Parity pin: every function reproduces the reference's double-precision operation order
 * (compiled with -ffp-contract=off, no -march, like the reference Release build) so that
 * tests/test_oracle_pin.py can require bit-identical results against the reference sources
 * compiled into oracle/_ref/libref_oracle.so, and against the golden fixtures in tests/golden/.
 * Reference file:line anchors are given per function (paths relative to /root/reference/proj).
 */
#include "oracle.h"

#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#define K_PI 3.14159265358979323846            /* vecmath.hpp:191 */
#define K_ALPHA_MIN (1.0 / 255.0)              /* rasterizer.hpp:18 */
#define K_ALPHA_MAX 0.99                       /* rasterizer.hpp:19 */
#define K_T_STOP 1e-4                          /* rasterizer.hpp:20 */
#define K_LOWPASS 0.3                          /* rasterizer.hpp:21 */
#define K_NEAR 0.01                            /* rasterizer.hpp:22 */
#define K_TILE 16                              /* rasterizer.hpp:23 */
#define K_POLE 1e-4                            /* camera.hpp:74 */
#define K_SH_C0 0.28209479177387814            /* scene.hpp:60 */

static const double kShC1 = 0.4886025119029199; /* scene.cpp:36-41 */
static const double kShC2[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005,
                                -1.0925484305920792, 0.5462742152960396};
static const double kShC3[7] = {-0.5900435899266435, 2.890611442640554, -0.4570457994644658,
                                0.3731763325901154, -0.4570457994644658, 1.445305721320277,
                                -0.5900435899266435};

static double g_last_seconds = 0.0;
static double now_s(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return ts.tv_sec + 1e-9 * ts.tv_nsec;
}

/* ------------------------------------------------------------------ small math (vecmath.hpp) */

static double dot3(const double* a, const double* b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }

/* Mat3 * Vec3, row-major (vecmath.hpp:84-88). */
static void m3v(const double* m, const double* v, double* o) {
    double r0 = m[0] * v[0] + m[1] * v[1] + m[2] * v[2];
    double r1 = m[3] * v[0] + m[4] * v[1] + m[5] * v[2];
    double r2 = m[6] * v[0] + m[7] * v[1] + m[8] * v[2];
    o[0] = r0; o[1] = r1; o[2] = r2;
}
/* M^T v (vecmath.hpp:115-119). */
static void m3tv(const double* m, const double* v, double* o) {
    double r0 = m[0] * v[0] + m[3] * v[1] + m[6] * v[2];
    double r1 = m[1] * v[0] + m[4] * v[1] + m[7] * v[2];
    double r2 = m[2] * v[0] + m[5] * v[1] + m[8] * v[2];
    o[0] = r0; o[1] = r1; o[2] = r2;
}
/* Mat23 (this) * R, accumulation from 0.0 in k order (vecmath.hpp:140-149). */
static void m23_mul(const double* a, const double* r, double* o) {
    for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 3; ++j) {
            double s = 0.0;
            for (int k = 0; k < 3; ++k) s += a[i * 3 + k] * r[k * 3 + j];
            o[i * 3 + j] = s;
        }
}
/* Quaternion (w,x,y,z) -> rotation (vecmath.hpp:171-184). */
static void quat_rot(const double* q, double* r) {
    double w = q[0], x = q[1], y = q[2], z = q[3];
    r[0] = 1 - 2 * (y * y + z * z);
    r[1] = 2 * (x * y - w * z);
    r[2] = 2 * (x * z + w * y);
    r[3] = 2 * (x * y + w * z);
    r[4] = 1 - 2 * (x * x + z * z);
    r[5] = 2 * (y * z - w * x);
    r[6] = 2 * (x * z - w * y);
    r[7] = 2 * (y * z + w * x);
    r[8] = 1 - 2 * (x * x + y * y);
}
static double qnorm(const double* q) { return sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]); }
static void qnormalize(const double* q, double* o) { /* vecmath.hpp:186-189 */
    double n = qnorm(q);
    o[0] = q[0] / n; o[1] = q[1] / n; o[2] = q[2] / n; o[3] = q[3] / n;
}

/* Sigma = R diag(s^2) R^T with normalized q, full 3x3 symmetric (scene.cpp:94-102). */
static void covariance3d(const double* q, const double* s, double* sig) {
    double qu[4], r[9];
    qnormalize(q, qu);
    quat_rot(qu, r);
    double s2[3] = {s[0] * s[0], s[1] * s[1], s[2] * s[2]};
    double full[9];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            double acc = 0.0;
            for (int k = 0; k < 3; ++k) acc += r[i * 3 + k] * s2[k] * r[j * 3 + k];
            full[i * 3 + j] = acc;
        }
    /* SymMat3 keeps the upper triangle and mirrors it (scene.hpp:16-28). */
    sig[0] = full[0]; sig[1] = full[1]; sig[2] = full[2];
    sig[3] = full[1]; sig[4] = full[4]; sig[5] = full[5];
    sig[6] = full[2]; sig[7] = full[5]; sig[8] = full[8];
}

/* Real SH basis, 3DGS sign convention (scene.cpp:45-67). */
static void sh_basis(const double* d, int degree, double* b) {
    b[0] = K_SH_C0;
    if (degree < 1) return;
    double x = d[0], y = d[1], z = d[2];
    b[1] = -kShC1 * y;
    b[2] = kShC1 * z;
    b[3] = -kShC1 * x;
    if (degree < 2) return;
    double xx = x * x, yy = y * y, zz = z * z;
    b[4] = kShC2[0] * x * y;
    b[5] = kShC2[1] * y * z;
    b[6] = kShC2[2] * (2.0 * zz - xx - yy);
    b[7] = kShC2[3] * x * z;
    b[8] = kShC2[4] * (xx - yy);
    if (degree < 3) return;
    b[9] = kShC3[0] * y * (3.0 * xx - yy);
    b[10] = kShC3[1] * x * y * z;
    b[11] = kShC3[2] * y * (4.0 * zz - xx - yy);
    b[12] = kShC3[3] * z * (2.0 * zz - 3.0 * xx - 3.0 * yy);
    b[13] = kShC3[4] * x * (4.0 * zz - xx - yy);
    b[14] = kShC3[5] * z * (xx - yy);
    b[15] = kShC3[6] * x * (xx - 3.0 * yy);
}

/* Basis gradients w.r.t. the direction components (scene.cpp:69-92). g is 16 x 3. */
static void sh_basis_grad(const double* d, int degree, double* b, double* g) {
    sh_basis(d, degree, b);
    g[0] = 0; g[1] = 0; g[2] = 0;
    if (degree < 1) return;
    double x = d[0], y = d[1], z = d[2];
#define SETG(i, a, bb, c) do { g[(i) * 3 + 0] = (a); g[(i) * 3 + 1] = (bb); g[(i) * 3 + 2] = (c); } while (0)
    SETG(1, 0, -kShC1, 0);
    SETG(2, 0, 0, kShC1);
    SETG(3, -kShC1, 0, 0);
    if (degree < 2) return;
    double xx = x * x, yy = y * y, zz = z * z;
    SETG(4, kShC2[0] * y, kShC2[0] * x, 0);
    SETG(5, 0, kShC2[1] * z, kShC2[1] * y);
    SETG(6, -2.0 * kShC2[2] * x, -2.0 * kShC2[2] * y, 4.0 * kShC2[2] * z);
    SETG(7, kShC2[3] * z, 0, kShC2[3] * x);
    SETG(8, 2.0 * kShC2[4] * x, -2.0 * kShC2[4] * y, 0);
    if (degree < 3) return;
    SETG(9, kShC3[0] * 6.0 * x * y, kShC3[0] * (3.0 * xx - 3.0 * yy), 0);
    SETG(10, kShC3[1] * y * z, kShC3[1] * x * z, kShC3[1] * x * y);
    SETG(11, -2.0 * kShC3[2] * x * y, kShC3[2] * (4.0 * zz - xx - 3.0 * yy), 8.0 * kShC3[2] * y * z);
    SETG(12, -6.0 * kShC3[3] * x * z, -6.0 * kShC3[3] * y * z, kShC3[3] * (6.0 * zz - 3.0 * xx - 3.0 * yy));
    SETG(13, kShC3[4] * (4.0 * zz - 3.0 * xx - yy), -2.0 * kShC3[4] * x * y, 8.0 * kShC3[4] * x * z);
    SETG(14, 2.0 * kShC3[5] * x * z, -2.0 * kShC3[5] * y * z, kShC3[5] * (xx - yy));
    SETG(15, kShC3[6] * (3.0 * xx - 3.0 * yy), -6.0 * kShC3[6] * x * y, 0);
#undef SETG
}

/* ------------------------------------------------------------------ camera (camera.cpp) */

/* dp/dt, Eqs. 11-16 (camera.cpp:52-68); caller has already rejected the pole. */
static void jacobian(const double* t, double t_r, int W, int H, double* j) {
    double tx = t[0], ty = t[1], tz = t[2];
    double u = tx * tx + tz * tz;
    double rho = sqrt(u);
    double r2 = t_r * t_r;
    double wf = W / (2.0 * K_PI);
    double hf = H / K_PI;
    j[0] = wf * tz / u;
    j[1] = 0.0;
    j[2] = -wf * tx / u;
    j[3] = -hf * tx * ty / (r2 * rho);
    j[4] = hf * rho / r2;
    j[5] = -hf * tz * ty / (r2 * rho);
}

/* dJ_rc/dt (camera.cpp:70-107); g[(r*3+c)*3 + k]. */
static void jacobian_grad(const double* t, double t_r, int W, int H, double* g) {
    double tx = t[0], ty = t[1], tz = t[2];
    double u = tx * tx + tz * tz;
    double rho = sqrt(u);
    double r2 = t_r * t_r;
    double u2 = u * u;
    double wf = W / (2.0 * K_PI);
    double hf = H / K_PI;
    double* g00 = g + 0; double* g01 = g + 3; double* g02 = g + 6;
    double* g10 = g + 9; double* g11 = g + 12; double* g12 = g + 15;
    g00[0] = -2.0 * wf * tx * tz / u2; g00[1] = 0.0; g00[2] = wf * (tx * tx - tz * tz) / u2;
    g01[0] = 0.0; g01[1] = 0.0; g01[2] = 0.0;
    g02[0] = wf * (tx * tx - tz * tz) / u2; g02[1] = 0.0; g02[2] = 2.0 * wf * tx * tz / u2;
    double base = hf / (r2 * rho);
    g10[0] = -base * ty * (1.0 - 2.0 * tx * tx / r2 - tx * tx / u);
    g10[1] = -base * tx * (1.0 - 2.0 * ty * ty / r2);
    g10[2] = base * tx * ty * tz * (2.0 / r2 + 1.0 / u);
    g11[0] = base * tx * (1.0 - 2.0 * u / r2);
    g11[1] = -2.0 * hf * rho * ty / (r2 * r2);
    g11[2] = base * tz * (1.0 - 2.0 * u / r2);
    g12[0] = base * tx * ty * tz * (2.0 / r2 + 1.0 / u);
    g12[1] = -base * tz * (1.0 - 2.0 * ty * ty / r2);
    g12[2] = -base * ty * (1.0 - 2.0 * tz * tz / r2 - tz * tz / u);
}

/* ------------------------------------------------------------------ rasterizer */

typedef struct proj {
    int gaussian_id;
    double p[2];
    double cov[3];   /* a, b, c */
    double conic[3];
    double radius, depth;
    double color[3];
    double alpha_base;
    double t[3];
} proj;

struct oracle_frame {
    int width, height;
    int nproj;
    proj* projections;
    int tiles_x, tiles_y;
    long* offsets; /* tiles + 1 */
    int* items;
    double* rgb;
    double* T;
    int* contrib;
    int* last;
    double background[3];
    int cloud_size;
    double pose[12];
};

static int bc_of(int degree) { return (degree + 1) * (degree + 1); }

/* project_gaussian (rasterizer.cpp:17-55). Returns 1 when visible. */
static int project_one(const oracle_cloud* c, int i, const double* pose, int W, int H, proj* out) {
    const double* R = pose;
    const double* tcw = pose + 9;
    double t[3];
    m3v(R, c->positions + 3 * i, t); /* world_to_camera (camera.cpp:21-23) */
    t[0] = t[0] + tcw[0]; t[1] = t[1] + tcw[1]; t[2] = t[2] + tcw[2];
    double t_r = sqrt(t[0] * t[0] + t[1] * t[1] + t[2] * t[2]);
    if (t_r < K_NEAR) return 0;
    double rho = sqrt(t[0] * t[0] + t[2] * t[2]);
    if (rho <= K_POLE * t_r) return 0;
    double opacity = 1.0 / (1.0 + exp(-c->opacity_logits[i])); /* scene.hpp:48-50 */
    if (opacity < K_ALPHA_MIN) return 0;

    /* project_equirect (camera.cpp:25-39) */
    double lon = atan2(t[0], t[2]);
    if (lon >= K_PI) lon -= 2.0 * K_PI;
    double sine = t[1] / t_r;
    sine = sine < -1.0 ? -1.0 : (sine > 1.0 ? 1.0 : sine);
    double lat = asin(sine);
    double sx = lon / K_PI, sy = 2.0 * lat / K_PI;
    out->p[0] = (sx + 1.0) * W * 0.5;
    out->p[1] = (sy + 1.0) * H * 0.5;

    double j[6], m[6];
    jacobian(t, t_r, W, H, j);
    m23_mul(j, R, m);
    double s[3] = {exp(c->log_scales[3 * i + 0]), exp(c->log_scales[3 * i + 1]),
                   exp(c->log_scales[3 * i + 2])};
    double s3[9];
    covariance3d(c->rotations + 4 * i, s, s3);
    double sm0[3], sm1[3];
    m3v(s3, m, sm0);
    m3v(s3, m + 3, sm1);
    double a = dot3(m, sm0) + K_LOWPASS;
    double b = dot3(m, sm1);
    double cc = dot3(m + 3, sm1) + K_LOWPASS;
    out->cov[0] = a; out->cov[1] = b; out->cov[2] = cc;
    double det = a * cc - b * b; /* SymMat2::inverse (vecmath.hpp:163-166) */
    out->conic[0] = cc / det; out->conic[1] = -b / det; out->conic[2] = a / det;
    double mid = 0.5 * (a + cc); /* SymMat2::max_eigenvalue (vecmath.hpp:158-162) */
    double dd = 0.25 * (a - cc) * (a - cc) + b * b;
    double d = sqrt(dd > 0.0 ? dd : 0.0);
    out->radius = ceil(3.0 * sqrt(mid + d));
    out->depth = t_r;
    out->alpha_base = opacity;
    out->t[0] = t[0]; out->t[1] = t[1]; out->t[2] = t[2];
    out->gaussian_id = i;

    /* view direction and eval_sh (rasterizer.cpp:51-53, scene.cpp:104-112) */
    double dir[3];
    m3tv(R, t, dir);
    double inv = 1.0 / t_r;
    dir[0] = dir[0] * inv; dir[1] = dir[1] * inv; dir[2] = dir[2] * inv;
    double basis[16];
    int deg = c->active_sh_degree;
    sh_basis(dir, deg, basis);
    int nb = bc_of(deg);
    const double* co = c->sh + (size_t)i * bc_of(c->sh_degree) * 3;
    double col[3] = {0, 0, 0};
    for (int k = 0; k < nb; ++k) {
        col[0] += co[3 * k + 0] * basis[k];
        col[1] += co[3 * k + 1] * basis[k];
        col[2] += co[3 * k + 2] * basis[k];
    }
    col[0] += 0.5; col[1] += 0.5; col[2] += 0.5;
    out->color[0] = col[0] > 0.0 ? col[0] : 0.0; /* std::max(0.0, x) */
    out->color[1] = col[1] > 0.0 ? col[1] : 0.0;
    out->color[2] = col[2] > 0.0 ? col[2] : 0.0;
    return 1;
}

static const proj* g_sort_proj; /* qsort context (single-threaded oracle) */
static int cmp_depth_id(const void* pa, const void* pb) {
    const proj* a = &g_sort_proj[*(const int*)pa];
    const proj* b = &g_sort_proj[*(const int*)pb];
    if (a->depth != b->depth) return a->depth < b->depth ? -1 : 1;
    return (a->gaussian_id > b->gaussian_id) - (a->gaussian_id < b->gaussian_id);
}

/* bin_to_tiles (rasterizer.cpp:57-98): inclusive floor bounds, pole clamp rows,
 * modulo-tiles_x seam wrap with the span >= tiles_x whole-row rule, per-tile (depth, id) sort. */
static void bin_tiles(oracle_frame* f) {
    const int tx_n = (f->width + K_TILE - 1) / K_TILE;
    const int ty_n = (f->height + K_TILE - 1) / K_TILE;
    const int tiles = tx_n * ty_n;
    f->tiles_x = tx_n;
    f->tiles_y = ty_n;
    long* count = (long*)calloc((size_t)tiles + 1, sizeof(long));
    /* two passes: count, then fill in projection order (== the reference push_back order) */
    for (int pass = 0; pass < 2; ++pass) {
        long* cursor = NULL;
        if (pass == 1) {
            f->offsets = (long*)malloc(((size_t)tiles + 1) * sizeof(long));
            f->offsets[0] = 0;
            for (int t = 0; t < tiles; ++t) f->offsets[t + 1] = f->offsets[t] + count[t];
            f->items = (int*)malloc((size_t)(f->offsets[tiles] > 0 ? f->offsets[tiles] : 1) * sizeof(int));
            cursor = (long*)malloc((size_t)tiles * sizeof(long));
            for (int t = 0; t < tiles; ++t) cursor[t] = f->offsets[t];
        }
        for (int i = 0; i < f->nproj; ++i) {
            const proj* pr = &f->projections[i];
            double y0 = pr->p[1] - pr->radius, y1 = pr->p[1] + pr->radius;
            int ty0 = (int)floor(y0 / K_TILE);
            if (ty0 < 0) ty0 = 0;
            int ty1 = (int)floor(y1 / K_TILE);
            if (ty1 > ty_n - 1) ty1 = ty_n - 1;
            if (ty0 > ty1) continue;
            int tx0 = (int)floor((pr->p[0] - pr->radius) / K_TILE);
            int tx1 = (int)floor((pr->p[0] + pr->radius) / K_TILE);
            if (tx1 - tx0 + 1 >= tx_n) { tx0 = 0; tx1 = tx_n - 1; }
            for (int ty = ty0; ty <= ty1; ++ty)
                for (int k = tx0; k <= tx1; ++k) {
                    int tx = ((k % tx_n) + tx_n) % tx_n;
                    int tile = ty * tx_n + tx;
                    if (pass == 0) count[tile]++;
                    else f->items[cursor[tile]++] = i;
                }
        }
        free(cursor);
    }
    free(count);
    g_sort_proj = f->projections;
    for (int t = 0; t < tiles; ++t) {
        long lo = f->offsets[t], hi = f->offsets[t + 1];
        if (hi - lo > 1) qsort(f->items + lo, (size_t)(hi - lo), sizeof(int), cmp_depth_id);
    }
}

/* One (pixel, splat) evaluation shared by blend and backward (rasterizer.cpp:128-134,
 * gradients.cpp:125-132). Returns 0 when the pair is skipped. */
static int eval_pair(const proj* pr, double sx, double sy, double width, double* dx_o, double* dy_o,
                     double* g_o, double* alpha_o) {
    double dx = remainder(pr->p[0] - sx, width);
    double dy = pr->p[1] - sy;
    double power = 0.5 * (pr->conic[0] * dx * dx + pr->conic[2] * dy * dy) + pr->conic[1] * dx * dy;
    if (power < 0.0) return 0;
    double g = exp(-power);
    double ab = pr->alpha_base * g;
    double alpha = ab < K_ALPHA_MAX ? ab : K_ALPHA_MAX; /* std::min(kAlphaMax, x) */
    if (alpha < K_ALPHA_MIN) return 0;
    *dx_o = dx; *dy_o = dy; *g_o = g; *alpha_o = alpha;
    return 1;
}

static oracle_frame* frame_new(const oracle_cloud* c, const double* pose, int W, int H, const double* bg) {
    oracle_frame* f = (oracle_frame*)calloc(1, sizeof(oracle_frame));
    f->width = W; f->height = H;
    f->cloud_size = c->n;
    memcpy(f->pose, pose, sizeof(double) * 12);
    for (int k = 0; k < 3; ++k) f->background[k] = bg ? bg[k] : 0.0;
    size_t px = (size_t)W * H;
    f->rgb = (double*)calloc(px * 3, sizeof(double));
    f->T = (double*)malloc(px * sizeof(double));
    f->contrib = (int*)calloc(px, sizeof(int));
    f->last = (int*)calloc(px, sizeof(int));
    for (size_t i = 0; i < px; ++i) f->T[i] = 1.0;
    f->projections = (proj*)malloc(((size_t)c->n + 1) * sizeof(proj));
    for (int i = 0; i < c->n; ++i)
        if (project_one(c, i, pose, W, H, &f->projections[f->nproj])) f->nproj++;
    return f;
}

/* blend_forward (rasterizer.cpp:100-157). */
static void blend(oracle_frame* f) {
    const int W = f->width, H = f->height;
    const double width = W;
    for (int ti = 0; ti < f->tiles_x * f->tiles_y; ++ti) {
        int tx = ti % f->tiles_x, ty = ti / f->tiles_x;
        int x0 = tx * K_TILE, x1 = x0 + K_TILE < W ? x0 + K_TILE : W;
        int y0 = ty * K_TILE, y1 = y0 + K_TILE < H ? y0 + K_TILE : H;
        long lo = f->offsets[ti], hi = f->offsets[ti + 1];
        for (int py = y0; py < y1; ++py)
            for (int px = x0; px < x1; ++px) {
                double sx = px + 0.5, sy = py + 0.5;
                double t_acc = 1.0, c[3] = {0, 0, 0};
                int contribs = 0, last = 0;
                for (long k = lo; k < hi; ++k) {
                    const proj* pr = &f->projections[f->items[k]];
                    double dx, dy, g, alpha;
                    if (!eval_pair(pr, sx, sy, width, &dx, &dy, &g, &alpha)) continue;
                    double t_next = t_acc * (1.0 - alpha);
                    if (t_next < K_T_STOP) break;
                    double w = alpha * t_acc;
                    c[0] += pr->color[0] * w; c[1] += pr->color[1] * w; c[2] += pr->color[2] * w;
                    t_acc = t_next;
                    ++contribs;
                    last = (int)(k - lo) + 1;
                }
                size_t pix = (size_t)py * W + px;
                f->rgb[pix * 3 + 0] = c[0] + t_acc * f->background[0];
                f->rgb[pix * 3 + 1] = c[1] + t_acc * f->background[1];
                f->rgb[pix * 3 + 2] = c[2] + t_acc * f->background[2];
                f->T[pix] = t_acc;
                f->contrib[pix] = contribs;
                f->last[pix] = last;
            }
    }
}

oracle_frame* oracle_render(const oracle_cloud* c, const double pose[12], int W, int H, const double bg[3]) {
    if (!c || !pose || W < 1 || H < 1) return NULL;
    double t0 = now_s();
    oracle_frame* f = frame_new(c, pose, W, H, bg);
    bin_tiles(f);
    blend(f);
    g_last_seconds = now_s() - t0;
    return f;
}

/* reference_render (rasterizer.cpp:177-235): every splat at every pixel, global order. */
oracle_frame* oracle_reference_render(const oracle_cloud* c, const double pose[12], int W, int H,
                                      const double bg[3]) {
    if (!c || !pose || W < 1 || H < 1) return NULL;
    oracle_frame* f = frame_new(c, pose, W, H, bg);
    int* order = (int*)malloc(((size_t)f->nproj + 1) * sizeof(int));
    for (int i = 0; i < f->nproj; ++i) order[i] = i;
    g_sort_proj = f->projections;
    if (f->nproj > 1) qsort(order, (size_t)f->nproj, sizeof(int), cmp_depth_id);
    const double width = W;
    for (int py = 0; py < H; ++py)
        for (int px = 0; px < W; ++px) {
            double sx = px + 0.5, sy = py + 0.5;
            double t_acc = 1.0, c3[3] = {0, 0, 0};
            int contribs = 0;
            for (int k = 0; k < f->nproj; ++k) {
                const proj* pr = &f->projections[order[k]];
                double dx, dy, g, alpha;
                if (!eval_pair(pr, sx, sy, width, &dx, &dy, &g, &alpha)) continue;
                double t_next = t_acc * (1.0 - alpha);
                if (t_next < K_T_STOP) break;
                double w = alpha * t_acc;
                c3[0] += pr->color[0] * w; c3[1] += pr->color[1] * w; c3[2] += pr->color[2] * w;
                t_acc = t_next;
                ++contribs;
            }
            size_t pix = (size_t)py * W + px;
            f->rgb[pix * 3 + 0] = c3[0] + t_acc * f->background[0];
            f->rgb[pix * 3 + 1] = c3[1] + t_acc * f->background[1];
            f->rgb[pix * 3 + 2] = c3[2] + t_acc * f->background[2];
            f->T[pix] = t_acc;
            f->contrib[pix] = contribs;
        }
    free(order);
    /* reference_render leaves the grid empty */
    f->tiles_x = 0; f->tiles_y = 0;
    f->offsets = (long*)calloc(1, sizeof(long));
    f->items = (int*)malloc(sizeof(int));
    return f;
}

oracle_frame* oracle_blend_projections(int n, const int* gid, const double* p, const double* cov,
                                       const double* conic, const double* radius, const double* depth,
                                       const double* color, const double* alpha, int W, int H, const double bg[3],
                                       const long* offsets, const int* items) {
    if (n < 0 || W < 1 || H < 1) return NULL;
    oracle_frame* f = (oracle_frame*)calloc(1, sizeof(oracle_frame));
    f->width = W; f->height = H;
    for (int k = 0; k < 3; ++k) f->background[k] = bg ? bg[k] : 0.0;
    for (int k = 0; k < 12; ++k) f->pose[k] = (k == 0 || k == 4 || k == 8) ? 1.0 : 0.0;
    size_t px = (size_t)W * H;
    f->rgb = (double*)calloc(px * 3, sizeof(double));
    f->T = (double*)malloc(px * sizeof(double));
    f->contrib = (int*)calloc(px, sizeof(int));
    f->last = (int*)calloc(px, sizeof(int));
    for (size_t i = 0; i < px; ++i) f->T[i] = 1.0;
    f->nproj = n;
    f->projections = (proj*)calloc((size_t)n + 1, sizeof(proj));
    for (int i = 0; i < n; ++i) {
        proj* pr = &f->projections[i];
        pr->gaussian_id = gid ? gid[i] : i;
        for (int k = 0; k < 2; ++k) pr->p[k] = p[2 * i + k];
        for (int k = 0; k < 3; ++k) {
            pr->cov[k] = cov[3 * i + k];
            pr->conic[k] = conic[3 * i + k];
            pr->color[k] = color[3 * i + k];
        }
        pr->radius = radius[i];
        pr->depth = depth[i];
        pr->alpha_base = alpha[i];
    }
    if (!offsets) {
        bin_tiles(f);
    } else {
        f->tiles_x = (W + K_TILE - 1) / K_TILE;
        f->tiles_y = (H + K_TILE - 1) / K_TILE;
        const int tiles = f->tiles_x * f->tiles_y;
        f->offsets = (long*)malloc(((size_t)tiles + 1) * sizeof(long));
        memcpy(f->offsets, offsets, ((size_t)tiles + 1) * sizeof(long));
        f->items = (int*)malloc((size_t)(offsets[tiles] > 0 ? offsets[tiles] : 1) * sizeof(int));
        if (offsets[tiles] > 0) memcpy(f->items, items, (size_t)offsets[tiles] * sizeof(int));
    }
    blend(f);
    return f;
}

void oracle_frame_free(oracle_frame* f) {
    if (!f) return;
    free(f->projections); free(f->offsets); free(f->items);
    free(f->rgb); free(f->T); free(f->contrib); free(f->last);
    free(f);
}

int oracle_frame_num_projections(const oracle_frame* f) { return f ? f->nproj : 0; }

void oracle_frame_projections(const oracle_frame* f, int* gid, double* p, double* cov, double* conic,
                              double* radius, double* depth, double* color, double* alpha, double* t) {
    for (int i = 0; i < f->nproj; ++i) {
        const proj* pr = &f->projections[i];
        if (gid) gid[i] = pr->gaussian_id;
        for (int k = 0; k < 2; ++k) if (p) p[2 * i + k] = pr->p[k];
        for (int k = 0; k < 3; ++k) {
            if (cov) cov[3 * i + k] = pr->cov[k];
            if (conic) conic[3 * i + k] = pr->conic[k];
            if (color) color[3 * i + k] = pr->color[k];
            if (t) t[3 * i + k] = pr->t[k];
        }
        if (radius) radius[i] = pr->radius;
        if (depth) depth[i] = pr->depth;
        if (alpha) alpha[i] = pr->alpha_base;
    }
}

long oracle_frame_tile_count(const oracle_frame* f, int* tx, int* ty) {
    if (tx) *tx = f->tiles_x;
    if (ty) *ty = f->tiles_y;
    return f->offsets[f->tiles_x * f->tiles_y];
}

void oracle_frame_tile_lists(const oracle_frame* f, long* offsets, int* items) {
    int tiles = f->tiles_x * f->tiles_y;
    if (offsets) memcpy(offsets, f->offsets, ((size_t)tiles + 1) * sizeof(long));
    if (items) memcpy(items, f->items, (size_t)f->offsets[tiles] * sizeof(int));
}

void oracle_frame_pixels(const oracle_frame* f, double* rgb, double* T, int* contrib, int* last) {
    size_t px = (size_t)f->width * f->height;
    if (rgb) memcpy(rgb, f->rgb, px * 3 * sizeof(double));
    if (T) memcpy(T, f->T, px * sizeof(double));
    if (contrib) memcpy(contrib, f->contrib, px * sizeof(int));
    if (last) memcpy(last, f->last, px * sizeof(int));
}

/* ------------------------------------------------------------------ backward (gradients.cpp) */

typedef struct acc9 {
    double d_color[3];
    double d_opacity;
    double d_p[2];
    double da, db, dc;
} acc9;

/* dR/dq_k for a unit quaternion (gradients.cpp:62-68). */
static void quat_rotation_grad(const double* q, double out[4][9]) {
    double w = q[0], x = q[1], y = q[2], z = q[3];
    double g0[9] = {0, -2 * z, 2 * y, 2 * z, 0, -2 * x, -2 * y, 2 * x, 0};
    double g1[9] = {0, 2 * y, 2 * z, 2 * y, -4 * x, -2 * w, 2 * z, 2 * w, -4 * x};
    double g2[9] = {-4 * y, 2 * x, 2 * w, 2 * x, 0, 2 * z, -2 * w, 2 * z, -4 * y};
    double g3[9] = {-4 * z, -2 * w, 2 * x, 2 * w, -4 * z, 2 * y, 2 * x, 2 * y, 0};
    memcpy(out[0], g0, sizeof g0); memcpy(out[1], g1, sizeof g1);
    memcpy(out[2], g2, sizeof g2); memcpy(out[3], g3, sizeof g3);
}

static int backward_impl(const oracle_frame* f, const double* d_image, const oracle_cloud* c,
                         const double pose[12], int W, int H, oracle_grads* gb);

int oracle_backward(const oracle_frame* f, const double* d_image, const oracle_cloud* c,
                    const double pose[12], int W, int H, oracle_grads* gb) {
    double t0 = now_s();
    int rc = backward_impl(f, d_image, c, pose, W, H, gb);
    g_last_seconds = now_s() - t0;
    return rc;
}

static int backward_impl(const oracle_frame* f, const double* d_image, const oracle_cloud* c,
                         const double pose[12], int W, int H, oracle_grads* gb) {
    /* state checks (gradients.cpp:74-80): only the rotation is compared */
    if (f->cloud_size != c->n || f->width != W || f->height != H ||
        memcmp(f->pose, pose, sizeof(double) * 9) != 0)
        return 1;
    const int n = c->n, bc = bc_of(c->sh_degree);
    memset(gb->d_position, 0, sizeof(double) * 3 * n);
    memset(gb->d_sh, 0, sizeof(double) * 3 * (size_t)n * bc);
    memset(gb->d_rotation, 0, sizeof(double) * 4 * n);
    memset(gb->d_log_scale, 0, sizeof(double) * 3 * n);
    memset(gb->d_opacity_logit, 0, sizeof(double) * n);
    memset(gb->d_screen, 0, sizeof(double) * 2 * n);

    const int tiles = f->tiles_x * f->tiles_y;
    const double width = W;
    const double* bg = f->background;
    long M = f->offsets[tiles];
    acc9* tile_acc = (acc9*)calloc((size_t)(M > 0 ? M : 1), sizeof(acc9));

    /* pass 1: per tile, back to front (gradients.cpp:96-160) */
    for (int ti = 0; ti < tiles; ++ti) {
        long lo = f->offsets[ti], hi = f->offsets[ti + 1];
        if (hi == lo) continue;
        int tx = ti % f->tiles_x, ty = ti / f->tiles_x;
        int x0 = tx * K_TILE, x1 = x0 + K_TILE < W ? x0 + K_TILE : W;
        int y0 = ty * K_TILE, y1 = y0 + K_TILE < H ? y0 + K_TILE : H;
        for (int py = y0; py < y1; ++py)
            for (int px = x0; px < x1; ++px) {
                size_t pix = (size_t)py * W + px;
                int last = f->last[pix];
                if (last == 0) continue;
                double dl[3] = {d_image[pix * 3 + 0], d_image[pix * 3 + 1], d_image[pix * 3 + 2]};
                double bg_dot = dot3(bg, dl);
                const double t_final = f->T[pix];
                double t_acc = t_final;
                double sx = px + 0.5, sy = py + 0.5;
                double suffix[3] = {0, 0, 0}, last_color[3] = {0, 0, 0};
                double last_alpha = 0.0;
                for (int k = last - 1; k >= 0; --k) {
                    const proj* pr = &f->projections[f->items[lo + k]];
                    double dx, dy, g, alpha;
                    if (!eval_pair(pr, sx, sy, width, &dx, &dy, &g, &alpha)) continue;
                    t_acc /= 1.0 - alpha;
                    acc9* slot = &tile_acc[lo + k];
                    double w_blend = alpha * t_acc;
                    for (int q = 0; q < 3; ++q) slot->d_color[q] += dl[q] * w_blend;
                    for (int q = 0; q < 3; ++q)
                        suffix[q] = last_color[q] * last_alpha + suffix[q] * (1.0 - last_alpha);
                    double diff[3] = {pr->color[0] - suffix[0], pr->color[1] - suffix[1],
                                      pr->color[2] - suffix[2]};
                    double d_alpha = dot3(diff, dl) * t_acc;
                    d_alpha -= t_final / (1.0 - alpha) * bg_dot;
                    for (int q = 0; q < 3; ++q) last_color[q] = pr->color[q];
                    last_alpha = alpha;
                    if (pr->alpha_base * g < K_ALPHA_MAX) {
                        slot->d_opacity += g * d_alpha;
                        double d_power = -g * pr->alpha_base * d_alpha;
                        double qx = pr->conic[0] * dx + pr->conic[1] * dy;
                        double qy = pr->conic[1] * dx + pr->conic[2] * dy;
                        double dpx = d_power * qx, dpy = d_power * qy;
                        slot->d_p[0] += dpx;
                        slot->d_p[1] += dpy;
                        slot->da += d_power * 0.5 * dx * dx;
                        slot->db += d_power * dx * dy;
                        slot->dc += d_power * 0.5 * dy * dy;
                    }
                }
            }
    }

    /* pass 2: fixed-order reduction (gradients.cpp:164-169) */
    acc9* proj_acc = (acc9*)calloc((size_t)f->nproj + 1, sizeof(acc9));
    for (int ti = 0; ti < tiles; ++ti)
        for (long k = f->offsets[ti]; k < f->offsets[ti + 1]; ++k) {
            acc9* a = &proj_acc[f->items[k]];
            const acc9* b = &tile_acc[k];
            for (int q = 0; q < 3; ++q) a->d_color[q] += b->d_color[q];
            a->d_opacity += b->d_opacity;
            a->d_p[0] += b->d_p[0];
            a->d_p[1] += b->d_p[1];
            a->da += b->da; a->db += b->db; a->dc += b->dc;
        }
    free(tile_acc);

    /* pass 3: per projection chain rule (gradients.cpp:173-295) */
    const double* R = pose;
    for (int j = 0; j < f->nproj; ++j) {
        const proj* pr = &f->projections[j];
        const acc9* acc = &proj_acc[j];
        const int gid = pr->gaussian_id;

        double ds0 = acc->d_p[0] * W * 0.5, ds1 = acc->d_p[1] * H * 0.5;
        gb->d_screen[2 * gid + 0] = ds0;
        gb->d_screen[2 * gid + 1] = ds1;
        gb->screen_norm_sum[gid] += sqrt(ds0 * ds0 + ds1 * ds1);
        gb->screen_hits[gid] += 1;

        double o = pr->alpha_base;
        gb->d_opacity_logit[gid] = acc->d_opacity * o * (1.0 - o);

        const double* t = pr->t;
        double t_r = sqrt(t[0] * t[0] + t[1] * t[1] + t[2] * t[2]);
        double dir[3];
        m3tv(R, t, dir);
        double inv = 1.0 / t_r;
        dir[0] = dir[0] * inv; dir[1] = dir[1] * inv; dir[2] = dir[2] * inv;
        double basis[16], dbasis[48];
        int deg = c->active_sh_degree;
        sh_basis_grad(dir, deg, basis, dbasis);
        int active_n = bc_of(deg);
        const double* co = c->sh + (size_t)gid * bc * 3;
        double raw[3] = {0.5, 0.5, 0.5};
        for (int i = 0; i < active_n; ++i)
            for (int q = 0; q < 3; ++q) raw[q] += co[3 * i + q] * basis[i];
        double dlc[3];
        for (int q = 0; q < 3; ++q) dlc[q] = raw[q] < 0.0 ? 0.0 : acc->d_color[q];
        double d_dir[3] = {0, 0, 0};
        for (int i = 0; i < active_n; ++i) {
            for (int q = 0; q < 3; ++q) gb->d_sh[((size_t)gid * bc + i) * 3 + q] = dlc[q] * basis[i];
            double cdot = co[3 * i + 0] * dlc[0] + co[3 * i + 1] * dlc[1] + co[3 * i + 2] * dlc[2];
            for (int q = 0; q < 3; ++q) d_dir[q] += dbasis[3 * i + q] * cdot;
        }
        double dd = dot3(dir, d_dir);
        double d_m_sh[3];
        for (int q = 0; q < 3; ++q) d_m_sh[q] = (d_dir[q] - dir[q] * dd) * (1.0 / t_r);

        double jac[6];
        jacobian(t, t_r, W, H, jac);
        double d_t[3] = {jac[0] * acc->d_p[0] + jac[3] * acc->d_p[1],
                         jac[1] * acc->d_p[0] + jac[4] * acc->d_p[1],
                         jac[2] * acc->d_p[0] + jac[5] * acc->d_p[1]};

        double qa = pr->conic[0], qb = pr->conic[1], qc = pr->conic[2];
        double da = acc->da, db = 0.5 * acc->db, dc = acc->dc;
        double m00 = qa * da + qb * db, m01 = qa * db + qb * dc;
        double m10 = qb * da + qc * db, m11 = qb * db + qc * dc;
        double dca = -(m00 * qa + m01 * qb);
        double dcb = -(m00 * qb + m01 * qc);
        double dcc = -(m10 * qb + m11 * qc);

        double m23[6];
        m23_mul(jac, R, m23);
        double s[3] = {exp(c->log_scales[3 * gid + 0]), exp(c->log_scales[3 * gid + 1]),
                       exp(c->log_scales[3 * gid + 2])};
        double s3[9];
        covariance3d(c->rotations + 4 * gid, s, s3);
        const double* m0 = m23;
        const double* m1 = m23 + 3;
        double dsig[9];
        for (int r = 0; r < 3; ++r)
            for (int cc = 0; cc < 3; ++cc)
                dsig[r * 3 + cc] = dca * m0[r] * m0[cc] + dcb * (m0[r] * m1[cc] + m1[r] * m0[cc]) +
                                   dcc * m1[r] * m1[cc];
        double sm0[3], sm1[3];
        m3v(s3, m0, sm0);
        m3v(s3, m1, sm1);
        double dm[6];
        for (int q = 0; q < 3; ++q) {
            dm[q] = (sm0[q] * dca + sm1[q] * dcb) * 2.0;
            dm[3 + q] = (sm0[q] * dcb + sm1[q] * dcc) * 2.0;
        }
        double Rt[9];
        for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b) Rt[a * 3 + b] = R[b * 3 + a];
        double djac[6];
        m23_mul(dm, Rt, djac);
        double jg[18];
        jacobian_grad(t, t_r, W, H, jg);
        for (int r = 0; r < 2; ++r)
            for (int cc = 0; cc < 3; ++cc) {
                const double* gv = jg + (r * 3 + cc) * 3;
                double dj = djac[r * 3 + cc];
                d_t[0] += gv[0] * dj; d_t[1] += gv[1] * dj; d_t[2] += gv[2] * dj;
            }
        double dpos[3];
        m3tv(R, d_t, dpos);
        for (int q = 0; q < 3; ++q) gb->d_position[3 * gid + q] = dpos[q] + d_m_sh[q];

        const double* q_raw = c->rotations + 4 * gid;
        double q_unit[4], rot[9];
        qnormalize(q_raw, q_unit);
        quat_rot(q_unit, rot);
        double d_rot[9];
        for (int r = 0; r < 3; ++r)
            for (int cc = 0; cc < 3; ++cc) {
                double v = 0.0;
                for (int k = 0; k < 3; ++k) v += dsig[r * 3 + k] * rot[k * 3 + cc];
                d_rot[r * 3 + cc] = 2.0 * v * s[cc] * s[cc];
            }
        double rg[4][9];
        quat_rotation_grad(q_unit, rg);
        double dqu[4];
        for (int k = 0; k < 4; ++k) {
            double v = 0.0;
            for (int i = 0; i < 9; ++i) v += d_rot[i] * rg[k][i];
            dqu[k] = v;
        }
        double qn = qnorm(q_raw);
        double qdot = q_unit[0] * dqu[0] + q_unit[1] * dqu[1] + q_unit[2] * dqu[2] + q_unit[3] * dqu[3];
        for (int k = 0; k < 4; ++k) gb->d_rotation[4 * gid + k] = (dqu[k] - q_unit[k] * qdot) / qn;

        for (int k = 0; k < 3; ++k) {
            double rk[3] = {rot[0 * 3 + k], rot[1 * 3 + k], rot[2 * 3 + k]};
            double srk[3];
            m3v(dsig, rk, srk);
            double rr = dot3(rk, srk);
            gb->d_log_scale[3 * gid + k] = 2.0 * s[k] * rr * s[k];
        }
    }
    free(proj_acc);
    return 0;
}

/* ------------------------------------------------------------------ Adam (trainer.cpp) */

static void adam_update(double* param, double grad, double* m, double* v, double lr, double bias1,
                        double bias2) {
    /* trainer.cpp:128-139; (1 - beta) folded exactly like the constexpr expression */
    const double b1 = 0.9, b2 = 0.999, eps = 1e-15;
    *m = b1 * *m + (1.0 - b1) * grad;
    *v = b2 * *v + (1.0 - b2) * grad * grad;
    double mhat = *m / bias1;
    double vhat = *v / bias2;
    *param -= lr * mhat / (sqrt(vhat) + eps);
}

void oracle_adam_step(oracle_cloud* c, const oracle_grads* g, oracle_adam* st, const oracle_adam_cfg* cfg,
                      double extent, long iteration) {
    const double t0 = now_s();
    const int n = c->n, bc = bc_of(c->sh_degree);
    st->step += 1;
    double bias1 = 1.0 - pow(0.9, (double)st->step);
    double bias2 = 1.0 - pow(0.999, (double)st->step);
    double t = 1.0;
    if (cfg->iterations > 0) {
        t = (double)iteration / cfg->iterations;
        t = t < 0.0 ? 0.0 : (t > 1.0 ? 1.0 : t);
    }
    double lr_pos = exp((1.0 - t) * log(cfg->lr_position_init * extent) +
                        t * log(cfg->lr_position_final * extent));
    for (int i = 0; i < n; ++i) {
        for (int k = 0; k < 3; ++k)
            adam_update(&c->positions[3 * i + k], g->d_position[3 * i + k], &st->m_position[3 * i + k],
                        &st->v_position[3 * i + k], lr_pos, bias1, bias2);
        for (int b = 0; b < bc; ++b) {
            double lr = b == 0 ? cfg->lr_sh_dc : cfg->lr_sh_rest;
            size_t base = ((size_t)i * bc + b) * 3;
            for (int k = 0; k < 3; ++k)
                adam_update(&c->sh[base + k], g->d_sh[base + k], &st->m_sh[base + k], &st->v_sh[base + k],
                            lr, bias1, bias2);
        }
        for (int k = 0; k < 4; ++k)
            adam_update(&c->rotations[4 * i + k], g->d_rotation[4 * i + k], &st->m_rotation[4 * i + k],
                        &st->v_rotation[4 * i + k], cfg->lr_rotation, bias1, bias2);
        for (int k = 0; k < 3; ++k)
            adam_update(&c->log_scales[3 * i + k], g->d_log_scale[3 * i + k], &st->m_scale[3 * i + k],
                        &st->v_scale[3 * i + k], cfg->lr_scale, bias1, bias2);
        adam_update(&c->opacity_logits[i], g->d_opacity_logit[i], &st->m_opacity[i], &st->v_opacity[i],
                    cfg->lr_opacity, bias1, bias2);
    }
    g_last_seconds = now_s() - t0;
}

/* ------------------------------------------------------------------ loss (trainer.cpp, metrics.cpp) */

#define K_WIN 11
#define K_HALF 5

static void ssim_window(double* w) { /* metrics.cpp:17-27 */
    double sum = 0.0;
    for (int i = 0; i < K_WIN; ++i) {
        double d = i - K_HALF;
        w[i] = exp(-d * d / (2.0 * 1.5 * 1.5));
        sum += w[i];
    }
    for (int i = 0; i < K_WIN; ++i) w[i] /= sum;
}

/* zero-padded separable same-size convolution (metrics.cpp:30-55) */
static void conv_same(const double* src, int w, int h, double* tmp, double* dst, const double* kern) {
    for (int y = 0; y < h; ++y) {
        const double* row = src + (size_t)y * w;
        double* out = tmp + (size_t)y * w;
        for (int x = 0; x < w; ++x) {
            double acc = 0.0;
            int k0 = -K_HALF > -x ? -K_HALF : -x;
            int k1 = K_HALF < w - 1 - x ? K_HALF : w - 1 - x;
            for (int k = k0; k <= k1; ++k) acc += kern[k + K_HALF] * row[x + k];
            out[x] = acc;
        }
    }
    for (int y = 0; y < h; ++y) {
        int k0 = -K_HALF > -y ? -K_HALF : -y;
        int k1 = K_HALF < h - 1 - y ? K_HALF : h - 1 - y;
        double* out = dst + (size_t)y * w;
        for (int x = 0; x < w; ++x) {
            double acc = 0.0;
            for (int k = k0; k <= k1; ++k) acc += kern[k + K_HALF] * tmp[(size_t)(y + k) * w + x];
            out[x] = acc;
        }
    }
}

/* ssim_with_gradient (metrics.cpp:81-153) on interleaved H x W x 3 images. */
static double ssim_grad(const double* a, const double* b, int w, int h, double* grad) {
    const double C1 = 0.01 * 0.01, C2 = 0.03 * 0.03;
    double kern[K_WIN];
    ssim_window(kern);
    size_t n = (size_t)w * h;
    double* buf = (double*)malloc(sizeof(double) * n * 17);
    double *x = buf, *y = buf + n, *xx = buf + 2 * n, *yy = buf + 3 * n, *xy = buf + 4 * n, *tmp = buf + 5 * n;
    double *mx = buf + 6 * n, *my = buf + 7 * n, *sxx = buf + 8 * n, *syy = buf + 9 * n, *sxy = buf + 10 * n;
    double *gmu = buf + 11 * n, *gsxx = buf + 12 * n, *gsxy = buf + 13 * n;
    double *cmu = buf + 14 * n, *csxx = buf + 15 * n, *csxy = buf + 16 * n;
    double total = 0.0;
    for (int ch = 0; ch < 3; ++ch) {
        for (size_t i = 0; i < n; ++i) {
            x[i] = a[i * 3 + ch];
            y[i] = b[i * 3 + ch];
            xx[i] = x[i] * x[i];
            yy[i] = y[i] * y[i];
            xy[i] = x[i] * y[i];
        }
        conv_same(x, w, h, tmp, mx, kern);
        conv_same(y, w, h, tmp, my, kern);
        conv_same(xx, w, h, tmp, sxx, kern);
        conv_same(yy, w, h, tmp, syy, kern);
        conv_same(xy, w, h, tmp, sxy, kern);
        double channel_sum = 0.0;
        for (size_t i = 0; i < n; ++i) {
            double m_x = mx[i], m_y = my[i];
            double var_x = sxx[i] - m_x * m_x;
            double var_y = syy[i] - m_y * m_y;
            double cov = sxy[i] - m_x * m_y;
            double a1 = 2.0 * m_x * m_y + C1;
            double a2 = 2.0 * cov + C2;
            double b1 = m_x * m_x + m_y * m_y + C1;
            double b2 = var_x + var_y + C2;
            double denom = b1 * b2;
            channel_sum += (a1 * a2) / denom;
            if (grad) {
                double d_a1 = a2 / denom;
                double d_a2 = a1 / denom;
                double d_b1 = -(a1 * a2) / (b1 * denom);
                double d_b2 = -(a1 * a2) / (b2 * denom);
                gmu[i] = d_a1 * 2.0 * m_y + d_b1 * 2.0 * m_x + d_a2 * (-2.0 * m_y) + d_b2 * (-2.0 * m_x);
                gsxx[i] = d_b2;
                gsxy[i] = d_a2 * 2.0;
            }
        }
        total += channel_sum / (double)n;
        if (grad) {
            conv_same(gmu, w, h, tmp, cmu, kern);
            conv_same(gsxx, w, h, tmp, csxx, kern);
            conv_same(gsxy, w, h, tmp, csxy, kern);
            double inv_n = 1.0 / (3.0 * (double)n);
            for (size_t i = 0; i < n; ++i)
                grad[i * 3 + ch] = inv_n * (cmu[i] + 2.0 * x[i] * csxx[i] + y[i] * csxy[i]);
        }
    }
    free(buf);
    return total / 3.0;
}

double oracle_loss(const double* r, const double* gt, int w, int h, double lambda, double mask_frac,
                   double* d_image) {
    const int masked = (int)floor(mask_frac * h);
    const int keep = h - masked;
    const size_t n = (size_t)w * keep * 3;
    double l1 = 0.0;
    double* d_l1 = (double*)malloc(sizeof(double) * (n + 1));
    for (size_t i = 0; i < n; ++i) {
        double d = r[i] - gt[i];
        l1 += fabs(d);
        d_l1[i] = d > 0.0 ? 1.0 : (d < 0.0 ? -1.0 : 0.0);
    }
    l1 /= (double)n;
    double value = (1.0 - lambda) * l1;
    double* d_ssim = NULL;
    if (lambda > 0.0) {
        d_ssim = (double*)calloc(n + 1, sizeof(double));
        double s = ssim_grad(r, gt, w, keep, d_ssim); /* the crop is the top `keep` rows */
        value += lambda * (1.0 - s);
    }
    if (d_image) {
        memset(d_image, 0, sizeof(double) * (size_t)w * h * 3);
        for (size_t i = 0; i < n; ++i) {
            double g = (1.0 - lambda) * d_l1[i] / (double)n;
            if (lambda > 0.0) g -= lambda * d_ssim[i];
            d_image[i] = g;
        }
    }
    free(d_l1);
    free(d_ssim);
    return value;
}

/* psnr (metrics.cpp:64-74, capped at kPsnrCap = 99) and ssim (metrics.cpp:76-79) — osplat_metrics
 * (capi.cpp:287-296). */
void oracle_metrics(const double* a, const double* b, int w, int h, double* psnr, double* ssim) {
    const size_t n = (size_t)w * h * 3;
    double mse = 0.0;
    for (size_t i = 0; i < n; ++i) {
        double d = a[i] - b[i];
        mse += d * d;
    }
    mse /= (double)n;
    if (psnr) {
        double v = 99.0;
        if (mse > 0.0) {
            v = 10.0 * log10(1.0 / mse);
            if (v > 99.0) v = 99.0;
        }
        *psnr = v;
    }
    if (ssim) *ssim = ssim_grad(a, b, w, h, NULL);
}

/* ------------------------------------------------------------------ densification (trainer.cpp) */

/* std::mt19937_64 (libstdc++ mersenne_twister_engine<uint64, 64, 312, 156, 31, 0xb5026f5aa96619e9,
 * 29, 0x5555555555555555, 17, 0x71d67fffeda60000, 37, 0xfff7eee000000000, 43, 6364136223846793005>). */
typedef struct {
    uint64_t x[312];
    int i;
} mt64;

static void mt64_seed(mt64* r, uint64_t seed) {
    r->x[0] = seed;
    for (int i = 1; i < 312; ++i) r->x[i] = 6364136223846793005ULL * (r->x[i - 1] ^ (r->x[i - 1] >> 62)) + (uint64_t)i;
    r->i = 312;
}

static uint64_t mt64_next(mt64* r) {
    if (r->i >= 312) {
        const uint64_t upper = ~0ULL << 31, lower = ~upper;
        for (int k = 0; k < 312; ++k) {
            uint64_t y = (r->x[k] & upper) | (r->x[(k + 1) % 312] & lower);
            r->x[k] = r->x[(k + 156) % 312] ^ (y >> 1) ^ ((y & 1ULL) ? 0xb5026f5aa96619e9ULL : 0ULL);
        }
        r->i = 0;
    }
    uint64_t z = r->x[r->i++];
    z ^= (z >> 29) & 0x5555555555555555ULL;
    z ^= (z << 17) & 0x71d67fffeda60000ULL;
    z ^= (z << 37) & 0xfff7eee000000000ULL;
    z ^= z >> 43;
    return z;
}

/* std::generate_canonical<double, 53>: one 64-bit draw scaled by 2^-64, clamped below 1. */
static double mt64_canonical(mt64* r) {
    double v = (double)mt64_next(r) / 18446744073709551616.0;
    return v >= 1.0 ? nextafter(1.0, 0.0) : v;
}

/* std::normal_distribution<double>(0, 1) in libstdc++: Marsaglia polar method, second value cached. */
typedef struct {
    mt64 eng;
    int saved_ok;
    double saved;
} normal_rng;

static double normal_next(normal_rng* g) {
    if (g->saved_ok) {
        g->saved_ok = 0;
        return g->saved;
    }
    double x, y, r2;
    do {
        x = 2.0 * mt64_canonical(&g->eng) - 1.0;
        y = 2.0 * mt64_canonical(&g->eng) - 1.0;
        r2 = x * x + y * y;
    } while (r2 > 1.0 || r2 == 0.0);
    const double mult = sqrt(-2 * log(r2) / r2);
    g->saved = x * mult;
    g->saved_ok = 1;
    return y * mult;
}

void oracle_mt64_draws(unsigned long long seed, long count, unsigned long long* out) {
    mt64 r;
    mt64_seed(&r, seed);
    for (long i = 0; i < count; ++i) out[i] = mt64_next(&r);
}

unsigned long long oracle_mix64(unsigned long long x) { /* trainer.cpp:300-306 */
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

static double max3(const double* v) { /* std::max({a, b, c}) */
    double m = v[0];
    if (m < v[1]) m = v[1];
    if (m < v[2]) m = v[2];
    return m;
}

static void copy_gaussian(const oracle_cloud* a, int i, const oracle_cloud* b, long j, int bc) {
    memcpy(b->positions + 3 * j, a->positions + 3 * (size_t)i, 3 * sizeof(double));
    memcpy(b->rotations + 4 * j, a->rotations + 4 * (size_t)i, 4 * sizeof(double));
    memcpy(b->log_scales + 3 * j, a->log_scales + 3 * (size_t)i, 3 * sizeof(double));
    b->opacity_logits[j] = a->opacity_logits[i];
    memcpy(b->sh + (size_t)j * bc * 3, a->sh + (size_t)i * bc * 3, (size_t)bc * 3 * sizeof(double));
}

/* densify_and_prune (trainer.cpp:188-275). The extended list is [originals | clones | split
 * children]; keep flags are decided on it and the survivors are compacted in order, together with
 * the Adam moments (AdamState::append_zeros + filter, trainer.cpp:100-124). */
int oracle_densify_and_prune(const oracle_cloud* in, const double* norm_sum, const long* hits,
                             const double* max_radius, const oracle_adam* st_in, const oracle_densify_cfg* cfg,
                             double extent, unsigned long long seed, int radius_active, oracle_cloud* out,
                             oracle_adam* st_out, oracle_edit* summary) {
    const double t0 = now_s();
    const int n = in->n, bc = bc_of(in->sh_degree);
    int* to_clone = (int*)malloc(sizeof(int) * (n > 0 ? n : 1));
    int* to_split = (int*)malloc(sizeof(int) * (n > 0 ? n : 1));
    long nc = 0, ns = 0;
    for (int i = 0; i < n; ++i) {
        const double g = hits[i] == 0 ? 0.0 : norm_sum[i] / (double)hits[i]; /* gradients.cpp:35-39 */
        if (g < cfg->densify_grad_threshold) continue;
        double s[3] = {exp(in->log_scales[3 * i]), exp(in->log_scales[3 * i + 1]), exp(in->log_scales[3 * i + 2])};
        if (max3(s) > cfg->scale_split_threshold * extent) to_split[ns++] = i;
        else to_clone[nc++] = i;
    }
    const long total = n + nc + 2 * ns;
    oracle_cloud ext = {(int)total, in->sh_degree, in->active_sh_degree,
                        (double*)malloc(sizeof(double) * 3 * total), (double*)malloc(sizeof(double) * 3 * bc * total),
                        (double*)malloc(sizeof(double) * 4 * total), (double*)malloc(sizeof(double) * 3 * total),
                        (double*)malloc(sizeof(double) * total)};
    char* keep = (char*)malloc(total > 0 ? total : 1);
    long* src = (long*)malloc(sizeof(long) * (total > 0 ? total : 1)); /* Adam source row, -1 = zeros */
    for (int i = 0; i < n; ++i) {
        copy_gaussian(in, i, &ext, i, bc);
        keep[i] = 1;
        src[i] = i;
    }
    long w = n;
    for (long k = 0; k < nc; ++k, ++w) {
        copy_gaussian(in, to_clone[k], &ext, w, bc);
        keep[w] = 1;
        src[w] = -1;
    }
    normal_rng rng;
    mt64_seed(&rng.eng, seed);
    rng.saved_ok = 0;
    const double log_split = log(cfg->split_factor);
    for (long k = 0; k < ns; ++k) {
        const int p = to_split[k];
        keep[p] = 0;
        double qn[4], rot[9];
        qnormalize(in->rotations + 4 * (size_t)p, qn);
        quat_rot(qn, rot);
        double s[3] = {exp(in->log_scales[3 * p]), exp(in->log_scales[3 * p + 1]), exp(in->log_scales[3 * p + 2])};
        for (int child = 0; child < 2; ++child, ++w) {
            double xi[3];
            xi[0] = normal_next(&rng) * s[0];
            xi[1] = normal_next(&rng) * s[1];
            xi[2] = normal_next(&rng) * s[2];
            copy_gaussian(in, p, &ext, w, bc);
            double d[3];
            m3v(rot, xi, d);
            for (int c = 0; c < 3; ++c) {
                ext.positions[3 * w + c] = in->positions[3 * (size_t)p + c] + d[c];
                ext.log_scales[3 * w + c] = in->log_scales[3 * (size_t)p + c] - log_split;
            }
            keep[w] = 1;
            src[w] = -1;
        }
    }
    /* prune (trainer.cpp:244-262) */
    long removed = 0;
    for (long i = 0; i < total; ++i) {
        if (keep[i]) {
            const double o = 1.0 / (1.0 + exp(-ext.opacity_logits[i]));
            double s[3] = {exp(ext.log_scales[3 * i]), exp(ext.log_scales[3 * i + 1]), exp(ext.log_scales[3 * i + 2])};
            if (o < cfg->prune_opacity) keep[i] = 0;
            else if (max3(s) > cfg->prune_scale_world * extent) keep[i] = 0;
            else if (radius_active && i < n && max_radius[i] > cfg->prune_radius_px) keep[i] = 0;
        }
        if (!keep[i]) ++removed;
    }
    long o = 0;
    for (long i = 0; i < total; ++i) {
        if (!keep[i]) continue;
        copy_gaussian(&ext, (int)i, out, o, bc);
#define ADAM_ROW(F, K)                                                                                  \
    if (src[i] >= 0) memcpy(st_out->F + (size_t)o * (K), st_in->F + (size_t)src[i] * (K), sizeof(double) * (K)); \
    else memset(st_out->F + (size_t)o * (K), 0, sizeof(double) * (K));
        ADAM_ROW(m_position, 3) ADAM_ROW(v_position, 3) ADAM_ROW(m_sh, 3 * bc) ADAM_ROW(v_sh, 3 * bc)
        ADAM_ROW(m_rotation, 4) ADAM_ROW(v_rotation, 4) ADAM_ROW(m_scale, 3) ADAM_ROW(v_scale, 3)
        ADAM_ROW(m_opacity, 1) ADAM_ROW(v_opacity, 1)
#undef ADAM_ROW
        ++o;
    }
    out->n = (int)o;
    out->sh_degree = in->sh_degree;
    out->active_sh_degree = in->active_sh_degree;
    st_out->step = st_in->step;
    summary->cloned = nc;
    summary->split = ns;
    summary->pruned = removed - ns;
    summary->final_count = o;
    free(ext.positions); free(ext.sh); free(ext.rotations); free(ext.log_scales); free(ext.opacity_logits);
    free(keep); free(src); free(to_clone); free(to_split);
    g_last_seconds = now_s() - t0;
    return 0;
}

void oracle_reset_opacity(oracle_cloud* c, double ceiling) { /* trainer.cpp:277-280 */
    const double cap = log(ceiling / (1.0 - ceiling));
    for (int i = 0; i < c->n; ++i)
        if (cap < c->opacity_logits[i]) c->opacity_logits[i] = cap;
}

void oracle_set_threads(int n) { (void)n; }
double oracle_last_seconds(void) { return g_last_seconds; }
int oracle_threads(void) { return 1; }
const char* oracle_kind(void) { return "port"; }
