/* oracle.h — TEST INFRASTRUCTURE ONLY (the parity checker, never the product).
 *
 * One C interface, two implementations:
 *   oracle/oracle.c      -> oracle/build/liboracle.so      (our FP64 C restatement)
 *   oracle/ref_shim.cpp  -> oracle/_ref/libref_oracle.so   (the reference's own C++ sources,
 *                                                           compiled from /root/reference)
 * Both export exactly these symbols so tests can diff them bit-for-bit.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg may load them.
 *
 * Layouts follow the reference GaussianCloud (proj/include/omnisplat/scene.hpp:31-55):
 *   positions  n x 3, sh n x bc x 3 (bc = (sh_degree+1)^2, RGB triples per basis function),
 *   rotations  n x 4 (w, x, y, z raw), log_scales n x 3, opacity_logits n.
 * Poses are 12 doubles: row-major 3x3 world->camera rotation, then translation
 * (proj/include/omnisplat/camera.hpp:21-30). */
#ifndef OSPLAT_ORACLE_H
#define OSPLAT_ORACLE_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct oracle_cloud {
    int n;
    int sh_degree;
    int active_sh_degree;
    double* positions;
    double* sh;
    double* rotations;
    double* log_scales;
    double* opacity_logits;
} oracle_cloud;

/* GradientBuffer (proj/include/omnisplat/gradients.hpp:16-36); caller-owned arrays. */
typedef struct oracle_grads {
    double* d_position;      /* n x 3 */
    double* d_sh;            /* n x bc x 3 */
    double* d_rotation;      /* n x 4 */
    double* d_log_scale;     /* n x 3 */
    double* d_opacity_logit; /* n */
    double* d_screen;        /* n x 2 */
    double* screen_norm_sum; /* n, accumulated across calls */
    long* screen_hits;       /* n, accumulated across calls */
} oracle_grads;

/* AdamState (proj/include/omnisplat/trainer.hpp:64-75), same flat layouts. */
typedef struct oracle_adam {
    double *m_position, *v_position;
    double *m_sh, *v_sh;
    double *m_rotation, *v_rotation;
    double *m_scale, *v_scale;
    double *m_opacity, *v_opacity;
    long step;
} oracle_adam;

/* The TrainConfig fields adam_step reads (proj/include/omnisplat/trainer.hpp:19-51). */
typedef struct oracle_adam_cfg {
    long iterations;
    double lr_position_init, lr_position_final;
    double lr_sh_dc, lr_sh_rest, lr_opacity, lr_scale, lr_rotation;
} oracle_adam_cfg;

typedef struct oracle_frame oracle_frame;

/* render(): project -> bin -> blend (proj/src/rasterizer.cpp:159-175). NULL on error. */
oracle_frame* oracle_render(const oracle_cloud* cloud, const double pose[12], int width, int height,
                            const double background[3]);
/* reference_render(): brute-force oracle (proj/src/rasterizer.cpp:177-235). */
oracle_frame* oracle_reference_render(const oracle_cloud* cloud, const double pose[12], int width,
                                      int height, const double background[3]);
void oracle_frame_free(oracle_frame* frame);
/* bin_to_tiles + blend_forward over n host SplatProjection records (rasterizer.cpp:57-157), arrays
 * as oracle_frame_projections (t unused). offsets == NULL: bin_to_tiles builds the grid; otherwise
 * offsets[tiles+1] / items[M] is the TileGrid to blend. */
oracle_frame* oracle_blend_projections(int n, const int* gaussian_id, const double* p, const double* cov,
                                       const double* conic, const double* radius, const double* depth,
                                       const double* color, const double* alpha_base, int width, int height,
                                       const double background[3], const long* offsets, const int* items);

int oracle_frame_num_projections(const oracle_frame* frame);
/* SplatProjection fields (proj/include/omnisplat/rasterizer.hpp:31-41); any pointer may be NULL. */
void oracle_frame_projections(const oracle_frame* frame, int* gaussian_id, double* p /*2*/,
                              double* cov /*3*/, double* conic /*3*/, double* radius,
                              double* depth, double* color /*3*/, double* alpha_base,
                              double* t /*3*/);
/* Tile grid: returns the instance count M. */
long oracle_frame_tile_count(const oracle_frame* frame, int* tiles_x, int* tiles_y);
/* CSR tile lists: offsets[tiles+1], items[M] = projection indices in blend order. */
void oracle_frame_tile_lists(const oracle_frame* frame, long* offsets, int* items);
/* RenderOutput pixel planes: rgb H x W x 3, T / contributors / last_contrib H x W. */
void oracle_frame_pixels(const oracle_frame* frame, double* rgb, double* transmittance,
                         int* contributors, int* last_contrib);

/* backward() (proj/src/gradients.cpp:72-296). Overwrites the gradients, accumulates the
 * screen statistics. Returns 0 on success, nonzero on StateMismatch. */
int oracle_backward(const oracle_frame* frame, const double* d_image, const oracle_cloud* cloud,
                    const double pose[12], int width, int height, oracle_grads* grads);

/* adam_step() (proj/src/trainer.cpp:143-178); mutates cloud and state. */
void oracle_adam_step(oracle_cloud* cloud, const oracle_grads* grads, oracle_adam* state,
                      const oracle_adam_cfg* cfg, double scene_extent, long iteration);

/* loss() (proj/src/trainer.cpp:25-71): (1-l)L1 + l(1-SSIM) with bottom-row masking.
 * d_image (H x W x 3) receives dL/dC; returns the loss value. */
double oracle_loss(const double* rendered, const double* gt, int width, int height,
                   double lambda_ssim, double mask_bottom_fraction, double* d_image);

/* psnr / ssim of two H x W x 3 images (metrics.cpp:64-79; osplat_metrics, capi.cpp:287-296). */
void oracle_metrics(const double* a, const double* b, int width, int height, double* psnr, double* ssim);

/* The TrainConfig fields densify_and_prune reads (proj/include/omnisplat/trainer.hpp:19-51). */
typedef struct oracle_densify_cfg {
    double densify_grad_threshold, scale_split_threshold, split_factor;
    double prune_opacity, prune_scale_world, prune_radius_px;
} oracle_densify_cfg;

/* EditSummary (proj/include/omnisplat/trainer.hpp:93-98). */
typedef struct oracle_edit {
    long cloned, split, pruned, final_count;
} oracle_edit;

/* densify_and_prune() (proj/src/trainer.cpp:188-275) on a cloud of n Gaussians with its screen
 * statistics (screen_norm_sum / screen_hits of the GradientBuffer), DensifyStats.max_radius_px and
 * AdamState; the rng is std::mt19937_64(rng_seed). The edited cloud / state are written to `out` /
 * `state_out`, whose arrays must hold 3n Gaussians (out->n is set). Returns 0. */
int oracle_densify_and_prune(const oracle_cloud* in, const double* screen_norm_sum, const long* screen_hits,
                             const double* max_radius_px, const oracle_adam* state_in,
                             const oracle_densify_cfg* cfg, double scene_extent, unsigned long long rng_seed,
                             int radius_prune_active, oracle_cloud* out, oracle_adam* state_out,
                             oracle_edit* summary);

/* reset_opacity() (proj/src/trainer.cpp:277-280): logits = min(logit, logit(ceiling)). */
void oracle_reset_opacity(oracle_cloud* cloud, double ceiling);

/* count raw draws of std::mt19937_64(seed) (Trainer::pick_view's shuffle, trainer.cpp:340-352). */
void oracle_mt64_draws(unsigned long long seed, long count, unsigned long long* out);

/* splitmix64 of the trainer's RNG streams (proj/src/trainer.cpp:300-306). */
unsigned long long oracle_mix64(unsigned long long x);

/* Reference-only file writers (ref_shim.cpp; not in the restatement): save_checkpoint
 * (dataio.cpp:347-382) and save_optimizer_state (dataio.cpp:479-495), for byte-level pins of the
 * product's PLY and OSPLADAM writers. Return 0 on success. */
int oracle_ref_save_checkpoint(const oracle_cloud* cloud, const char* path);
int oracle_ref_save_optimizer_state(const oracle_adam* state, int n, int basis_count, long iteration,
                                    const char* path);

/* Wall time (steady clock, like eval.cpp:84-87) of the last render / backward / adam_step / loss
 * call, excluding the marshalling between these flat arrays and the implementation's types. */
double oracle_last_seconds(void);

/* Thread count of the implementation (reference: OMNISPLAT_THREADS; restatement: 1). */
void oracle_set_threads(int n);
int oracle_threads(void);
const char* oracle_kind(void);

#ifdef __cplusplus
}
#endif

#endif
