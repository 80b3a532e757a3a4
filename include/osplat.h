/* osplat.h — C ABI of the B200-native ERP Gaussian-splatting hot path (libosplat_b200.so).
 *
 * Part 1 re-exports the reference C interface for this path with byte-identical signatures and
 * semantics (reference: /root/reference/proj/include/omnisplat/capi.h). Every call returns
 * osplat_status; on failure osplat_last_error() holds "<ErrorCode>: message" for the calling
 * thread (capi.cpp:39,68-81). Handles are opaque and freed with their _free function (NULL OK).
 *
 * Part 2 adds the device-resident render / backward / step interface the reference exposes only
 * in C++ (rasterizer.hpp:85-86 render, gradients.hpp:43-44 backward, trainer.hpp:80-81
 * adam_step), as plain-pointer C entry points. No torch or CUDA types appear in any signature;
 * streams and device buffers cross the boundary as void* / typed device pointers.
 *
 * Threading contract (same as the reference, SPEC.md exclusivity): an osplat_gpu context and the
 * frames it produced must not be used concurrently from two host threads. osplat_render may be
 * called from any number of threads on one osplat_cloud (the cloud is read-shared):
 * the cloud's device copy is created once and concurrent renders of it are serialised. Calls are ordered on
 * the context's CUDA stream; every call that returns host data synchronizes that stream.
 */
#ifndef OSPLAT_B200_H
#define OSPLAT_B200_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define OSPLAT_API __attribute__((visibility("default")))
#else
#define OSPLAT_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* ======================================================================================
 * Part 1 — reference C ABI (capi.h)
 * ====================================================================================== */

/* capi.h:15-23 */
typedef enum osplat_status {
    OSPLAT_OK = 0,
    OSPLAT_ERR_INVALID_ARGUMENT = 1,
    OSPLAT_ERR_IO = 2,
    OSPLAT_ERR_PARSE = 3,
    OSPLAT_ERR_VALIDATION = 4,
    OSPLAT_ERR_UNSUPPORTED = 5,
    OSPLAT_ERR_RUNTIME = 6
} osplat_status;

typedef struct osplat_cloud osplat_cloud;   /* capi.h:25 — host GaussianCloud (scene.hpp:31-55) */
typedef struct osplat_config osplat_config; /* capi.h:27 — TrainConfig (trainer.hpp:19-51) */
typedef struct osplat_image osplat_image;   /* capi.h:28 — H x W x 3 double image (image.hpp) */

OSPLAT_API const char* osplat_version(void);     /* capi.h:31 */
OSPLAT_API const char* osplat_last_error(void);  /* capi.h:33 */
/* capi.h:36 — accepted for compatibility; the GPU path has no CPU worker pool. */
OSPLAT_API void osplat_set_threads(int n);

/* capi.h:39-42 — checkpoint PLY (dataio.cpp:347-453 format: binary little-endian float32). */
OSPLAT_API osplat_status osplat_cloud_load(const char* path, osplat_cloud** out);
OSPLAT_API osplat_status osplat_cloud_save(const osplat_cloud* cloud, const char* path);
OSPLAT_API size_t osplat_cloud_count(const osplat_cloud* cloud);
OSPLAT_API void osplat_cloud_free(osplat_cloud* cloud);

/* capi.h:56-60 — training configuration (set_train_config_field keys, dataio.cpp:570-605). */
OSPLAT_API osplat_status osplat_config_create(osplat_config** out);
OSPLAT_API osplat_status osplat_config_set(osplat_config* config, const char* key, const char* value);
OSPLAT_API void osplat_config_free(osplat_config* config);

/* capi.h:73-74 — renders on the GPU (device OSPLAT_DEVICE, default 0), tile 16, black
 * background, the cloud's active SH degree; synchronous; *out owns an H x W x 3 double image. */
OSPLAT_API osplat_status osplat_render(const osplat_cloud* cloud, const double transform_cw[16], int width, int height,
                            osplat_image** out);

/* capi.h:84-88 */
OSPLAT_API int osplat_image_width(const osplat_image* image);
OSPLAT_API int osplat_image_height(const osplat_image* image);
OSPLAT_API const double* osplat_image_pixels(const osplat_image* image);
OSPLAT_API void osplat_image_free(osplat_image* image);

/* capi.h:90-92 — PSNR (dB, capped at 99) and SSIM (11x11, sigma 1.5, zero-padded; mean over pixels
 * and channels) of two images of equal size, computed in FP64 on the GPU (metrics.cpp:17-79).
 * Sizes differ -> OSPLAT_ERR_VALIDATION "DimensionMismatch: psnr: image sizes differ". Either
 * output pointer may be NULL. Synchronous. */
OSPLAT_API osplat_status osplat_metrics(const osplat_image* a, const osplat_image* b, double* out_psnr,
                                        double* out_ssim);

/* ======================================================================================
 * Part 2 — device-resident render / backward / step interface
 * ====================================================================================== */

/* Build a host cloud from reference-layout arrays (GaussianCloud fields, scene.hpp:35-39):
 * positions n*3, sh n*(sh_degree+1)^2*3, rotations n*4 (w,x,y,z), log_scales n*3, opacity n. */
OSPLAT_API osplat_status osplat_cloud_create(size_t n, int sh_degree, int active_sh_degree, const double* positions,
                                  const double* sh, const double* rotations, const double* log_scales,
                                  const double* opacity_logits, osplat_cloud** out);
/* Copy a host cloud back out (any pointer may be NULL). */
OSPLAT_API osplat_status osplat_cloud_read(const osplat_cloud* cloud, double* positions, double* sh, double* rotations,
                                double* log_scales, double* opacity_logits, int* sh_degree,
                                int* active_sh_degree);

typedef struct osplat_gpu osplat_gpu;     /* device context: parameters, gradients, Adam moments */
typedef struct osplat_frame osplat_frame; /* retained forward state of one render (RenderOutput) */

/* Create a context on `device`, ordering all work on `cuda_stream` (a cudaStream_t; NULL = the
 * context creates its own non-blocking stream), and upload `cloud` to FP32 SoA planes. */
OSPLAT_API osplat_status osplat_gpu_create(int device, void* cuda_stream, const osplat_cloud* cloud, osplat_gpu** out);
OSPLAT_API void osplat_gpu_free(osplat_gpu* ctx);
OSPLAT_API size_t osplat_gpu_count(const osplat_gpu* ctx);
OSPLAT_API osplat_status osplat_gpu_set_active_sh_degree(osplat_gpu* ctx, int degree);
/* Optional deterministic backward (the reference's pass 2 is a fixed-order tile reduction,
 * gradients.cpp:162-169, so its gradients do not depend on the schedule): on != 0 makes every
 * following backward of this context run K4a without atomics — per-instance partials, summed per
 * Gaussian in a fixed order — so gradients are bit-identical run to run. Default off (K4a's
 * warp-aggregated atomics: same values up to FP32 summation order, about half the cost). */
OSPLAT_API osplat_status osplat_gpu_set_deterministic(osplat_gpu* ctx, int on);
/* Verification mode of the blend's T < 1e-4 stop: on != 0 replaces the default
 * relative 2^-10 guard band by a running bound on the FP32 transmittance's error (built from K1's
 * per-Gaussian power bound), so every stop decision is provably the FP64 reference's; more pixels
 * replay in FP64 (slower). Frames of both modes are compared in tests/test_gpu_fullsize.py. */
OSPLAT_API osplat_status osplat_gpu_set_strict_guard(osplat_gpu* ctx, int on);
/* Download the current parameters into a new host cloud. */
OSPLAT_API osplat_status osplat_gpu_download(osplat_gpu* ctx, osplat_cloud** out);
OSPLAT_API osplat_status osplat_gpu_synchronize(osplat_gpu* ctx);

/* render (rasterizer.hpp:85-86): K1 preprocess -> K2 sort -> K3 blend. transform_cw is the
 * row-major 4x4 world->camera matrix (capi.cpp:88-95); background may be NULL (black). */
OSPLAT_API osplat_status osplat_gpu_render(osplat_gpu* ctx, const double transform_cw[16], int width, int height,
                                const double background[3], osplat_frame** out);
OSPLAT_API void osplat_frame_free(osplat_frame* frame);
OSPLAT_API int osplat_frame_width(const osplat_frame* frame);
OSPLAT_API int osplat_frame_height(const osplat_frame* frame);
/* Host copies of the RenderOutput pixel state (rasterizer.hpp:52-57); NULL pointers skipped.
 * rgb is H x W x 3 (interleaved, like Image), the rest H x W. */
OSPLAT_API osplat_status osplat_frame_image(const osplat_frame* frame, double* rgb);
OSPLAT_API osplat_status osplat_frame_pixels(const osplat_frame* frame, float* rgb, float* transmittance,
                                  int* contributors, int* last_contrib);
/* Per-Gaussian projection state indexed by Gaussian id (n entries): visible flag, FP64 centre
 * (2), FP64 conic (3), opacity, FP32 colour (3), tile rect {tx0,tx1,ty0,ty1} (4), instances. */
OSPLAT_API osplat_status osplat_frame_projections(const osplat_frame* frame, uint8_t* visible, double* p, double* conic,
                                       double* opacity, float* color, int32_t* rect, uint32_t* touched);
/* Sorted tile lists: *instances = M; ranges (2 per tile, [begin, end)) and gaussian ids (M).
 * Call with NULL arrays first to size them. */
OSPLAT_API osplat_status osplat_frame_tiles(const osplat_frame* frame, int* tiles_x, int* tiles_y, size_t* instances,
                                 uint32_t* ranges, uint32_t* gaussian_ids);

/* Full SplatProjection records (rasterizer.hpp:31-41) of a frame: the visible Gaussians in
 * ascending id (render()'s compaction, rasterizer.cpp:165-168), or for a frame of host projections
 * (osplat_gpu_render_projected) the records as given. Call with NULL arrays to get *count. Arrays
 * are per record: gaussian_id, p (2), cov (3), conic (3), radius, depth, color (3), alpha_base,
 * t (3; zeros for host projections). Colour is the FP32 value the blend uses. */
OSPLAT_API osplat_status osplat_frame_splats(const osplat_frame* frame, size_t* count, int32_t* gaussian_id,
                                             double* p, double* cov, double* conic, double* radius, double* depth,
                                             double* color, double* alpha_base, double* t);

/* Replace the context's cloud (GaussianCloud assignment; Adam state and statistics reset). */
OSPLAT_API osplat_status osplat_gpu_upload(osplat_gpu* ctx, const osplat_cloud* cloud);

/* bin_to_tiles + blend_forward (rasterizer.cpp:57-157) over `count` host SplatProjection records
 * (same per-record arrays as osplat_frame_splats; gaussian_id may be NULL = index; cov must be
 * conic^-1, as project_gaussian produces it). tile_offsets == NULL: the device bins and sorts the
 * records by (depth, gaussian_id) like bin_to_tiles (read the lists back with osplat_frame_tiles;
 * its ids are then record indices). Otherwise the caller's TileGrid is blended as given:
 * tile_offsets has tiles+1 entries (tiles = ceil(W/16) ceil(H/16)), tile_entries the concatenated
 * record indices. The frame has no Gaussian parameters behind it: osplat_gpu_backward on it fails
 * with a validation status (StateMismatch). Depth must be finite and >= 0. */
OSPLAT_API osplat_status osplat_gpu_render_projected(osplat_gpu* ctx, size_t count, const int32_t* gaussian_id,
                                                     const double* p, const double* cov, const double* conic,
                                                     const double* radius, const double* depth, const double* color,
                                                     const double* alpha_base, int width, int height,
                                                     const double background[3], const uint32_t* tile_offsets,
                                                     const int32_t* tile_entries, osplat_frame** out);

/* Device views for zero-copy interop (e.g. wrapping as torch tensors for NCCL). */
typedef struct osplat_frame_view {
    float* rgb;           /* 3 planes of H*W (R, G, B) */
    float* transmittance; /* H*W */
    int* contributors;    /* H*W */
    int* last_contrib;    /* H*W */
    int width, height;
} osplat_frame_view;
OSPLAT_API osplat_status osplat_frame_device(const osplat_frame* frame, osplat_frame_view* view);

typedef struct osplat_gpu_view {
    float* params;    /* planes * stride FP32: pos 3 | SH 3*bc | rot 4 | log-scale 3 | opacity 1 */
    float* grads;     /* same layout; the buffer NCCL allreduces */
    float* adam_m;
    float* adam_v;
    float* d_screen;  /* n * 2 */
    double* screen_norm_sum;
    int32_t* screen_hits;
    size_t n, stride;
    int planes, sh_degree, active_sh_degree;
    long adam_step;
    float* max_radius_px; /* n: DensifyStats.max_radius_px (trainer.hpp:85-91) */
} osplat_gpu_view;
OSPLAT_API osplat_status osplat_gpu_view_buffers(osplat_gpu* ctx, osplat_gpu_view* view);

/* backward (gradients.hpp:43-44). d_image is dL/dC: host H x W x 3 double (reference Image
 * layout) for osplat_gpu_backward, device planar FP32 (3 planes of H*W) for _device. With
 * accumulate = 0 the raw-parameter gradients are overwritten (reference semantics); with 1 they
 * are added (multi-view batches). Screen statistics always accumulate (GradientBuffer). */
OSPLAT_API osplat_status osplat_gpu_backward(osplat_gpu* ctx, const osplat_frame* frame, const double* d_image, int accumulate);
OSPLAT_API osplat_status osplat_gpu_backward_device(osplat_gpu* ctx, const osplat_frame* frame, const float* d_image_planar,
                                         int accumulate);
/* Raw-parameter gradients in reference GradientBuffer layout (gradients.hpp:16-36). */
OSPLAT_API osplat_status osplat_gpu_gradients(osplat_gpu* ctx, double* d_position, double* d_sh, double* d_rotation,
                                   double* d_log_scale, double* d_opacity_logit, double* d_screen,
                                   double* screen_norm_sum, long* screen_hits);
/* zero_grad: the gradient planes become logically zero without a memory pass — the next backward
 * stores instead of adding, and any read of the planes before that (osplat_gpu_gradients,
 * osplat_gpu_view_buffers, whose caller may hand the planes to a collective) writes real zeros
 * first. */
OSPLAT_API osplat_status osplat_gpu_zero_grad(osplat_gpu* ctx);
OSPLAT_API osplat_status osplat_gpu_reset_screen_stats(osplat_gpu* ctx);

/* adam_step (trainer.hpp:80-81): one fused launch over all planes; config may be NULL
 * (reference defaults). zero_grad != 0 leaves the consumed gradients logically zero (see
 * osplat_gpu_zero_grad). */
OSPLAT_API osplat_status osplat_gpu_adam_step(osplat_gpu* ctx, const osplat_config* config, double scene_extent,
                                   long iteration, int zero_grad);
/* The same step over the flat element range [begin, begin + count) of the planes x stride buffers
 * (multiples of 4): a data-parallel rank's shard after a reduce-scatter of the gradients, followed
 * by an all-gather of the parameters (sharded optimizer; every rank advances the step counter). */
OSPLAT_API osplat_status osplat_gpu_adam_step_range(osplat_gpu* ctx, const osplat_config* config, double scene_extent,
                                                    long iteration, int zero_grad, size_t begin, size_t count);

/* ---- evaluation (capi.h:94-105, run_eval eval.cpp:63-116) over in-memory views: views poses
 * (row-major 4x4 world->camera each) and images; is_test (NULL: none) marks the test split;
 * split "test" (default when NULL), "train" or "all"; perspective_crop != 0 evaluates on the 6
 * cube faces (H/2 x H/2, 90 degree FOV) of each panorama instead of the panorama. Render time per
 * view on the steady clock around the render and its completion (the reference's FPS convention);
 * PSNR / SSIM in FP64 on the device. Unknown split -> OSPLAT_ERR_INVALID_ARGUMENT, empty split ->
 * OSPLAT_ERR_VALIDATION (EmptySplit). */
typedef struct osplat_report osplat_report; /* capi.h — EvalReport (eval.hpp:28-35) */
OSPLAT_API osplat_status osplat_gpu_eval(osplat_gpu* ctx, size_t views, const double* transforms_cw,
                                         const osplat_image* const* images, const unsigned char* is_test,
                                         const char* split, int perspective_crop, osplat_report** out);
OSPLAT_API size_t osplat_report_view_count(const osplat_report* report);
OSPLAT_API osplat_status osplat_report_view(const osplat_report* report, size_t index, int* frame_index,
                                            double* psnr, double* ssim);
OSPLAT_API osplat_status osplat_report_mean(const osplat_report* report, double* psnr, double* ssim,
                                            double* seconds_per_frame, double* fps);
OSPLAT_API const char* osplat_report_mode(const osplat_report* report);
OSPLAT_API void osplat_report_free(osplat_report* report);

/* ---- §8(e) multi-view data parallelism inside the library: one process (context) per GPU, one
 * NCCL communicator per context, every collective issued by the library on the context stream.
 * NCCL is loaded at run time (libnccl.so.2; the one already mapped by the process if any; the
 * environment variable OSPLAT_NCCL_LIB names another library); without it these calls return
 * OSPLAT_ERR_UNSUPPORTED.
 * osplat_nccl_unique_id: ncclGetUniqueId on one rank; the launcher hands the 128 bytes to every
 * rank (any channel: torch.distributed, MPI, a file). osplat_gpu_dp_init: ncclCommInitRank
 * (collective over the world). osplat_gpu_dp_step: the batch's exchange + optimizer step after
 * every rank's backward(s) — in-place reduce-scatter of the gradient planes, fused Adam on this
 * rank's 1/world shard, in-place all-gather of the parameters (= allreduce + replicated Adam, with
 * 1/world of the Adam traffic; replicas bit-identical). With a communicator,
 * osplat_gpu_densify_and_prune sums the screen statistics and maxes the radii over ranks and
 * gathers the Adam moments first, osplat_gpu_save_state gathers the moments, and osplat_gpu_train
 * trains a batch of `world` views per iteration (entry (j-1) world + rank of the reference's view
 * stream on this rank; rank 0 writes the files): all of these are collectives — call them on
 * every rank. */
OSPLAT_API osplat_status osplat_nccl_unique_id(unsigned char id[128]);
OSPLAT_API osplat_status osplat_gpu_dp_init(osplat_gpu* ctx, int world, int rank, const unsigned char id[128]);
OSPLAT_API osplat_status osplat_gpu_dp_step(osplat_gpu* ctx, const osplat_config* config, double scene_extent,
                                            long iteration);

/* loss() (trainer.cpp:25-71): (1 - lambda_ssim) L1 + lambda_ssim (1 - SSIM), SSIM 11x11 sigma 1.5
 * zero-padded (metrics.cpp:17-153), bottom rows masked, against a device planar FP32 target:
 * writes dL/dC into the context's d_image buffer (returned through *d_image_planar) and the
 * loss value (host, synchronizes) into *loss unless loss is NULL. _l1_loss = lambda_ssim 0. */
OSPLAT_API osplat_status osplat_gpu_loss(osplat_gpu* ctx, const osplat_frame* frame, const float* gt_planar_device,
                                         double lambda_ssim, double mask_bottom_fraction,
                                         const float** d_image_planar, double* loss);
OSPLAT_API osplat_status osplat_gpu_l1_loss(osplat_gpu* ctx, const osplat_frame* frame, const float* gt_planar_device,
                                 double mask_bottom_fraction, const float** d_image_planar, double* loss);

/* One training view: render -> loss -> backward (accumulate) against `gt` (host or device
 * planar FP32, 3*H*W; a host target is uploaded on a side stream, overlapped with the render),
 * returning the loss in *loss (host) — the per-view part of Trainer::run (trainer.cpp:360-363).
 * The caller follows with osplat_gpu_adam_step. */
OSPLAT_API osplat_status osplat_gpu_train_view(osplat_gpu* ctx, const double transform_cw[16], int width, int height,
                                    const float* gt_planar, int gt_on_device, double lambda_ssim,
                                    double mask_bottom_fraction, double* loss);
/* osplat_gpu_train_view without the per-step wait: every kernel and copy of the step is enqueued on
 * the context's stream and the call returns. loss_sums (4 doubles, pinned host memory; may be NULL)
 * receives {L1 sum, SSIM sums r, g, b} once the stream reaches the end of the step — read them after
 * osplat_gpu_synchronize and turn them into the loss with osplat_loss_value. A pipelined training
 * loop (loss logged one step late) keeps the GPU busy while the host enqueues the next view.
 * A host target (gt_on_device 0) is copied asynchronously when it is page-locked: keep it valid
 * and unmodified until the stream has passed the step. */
OSPLAT_API osplat_status osplat_gpu_train_view_async(osplat_gpu* ctx, const double transform_cw[16], int width,
                                                     int height, const float* gt, int gt_on_device,
                                                     double lambda_ssim, double mask_bottom_fraction,
                                                     double* loss_sums);
/* (1 - l) L1 + l (1 - SSIM) from the sums of osplat_gpu_train_view_async (trainer.cpp:54-63). */
OSPLAT_API double osplat_loss_value(const double sums[4], double lambda_ssim, int width, int height,
                                    double mask_bottom_fraction);

/* ---- densification control (trainer.cpp:180-280) ---- */
/* EditSummary (trainer.hpp:93-98). */
typedef struct osplat_edit_summary {
    long cloned, split, pruned;
    size_t final_count;
} osplat_edit_summary;
/* DensifyStats::observe (trainer.cpp:180-186): per-Gaussian max screen radius over the frames
 * observed since the last densification. */
OSPLAT_API osplat_status osplat_gpu_observe(osplat_gpu* ctx, const osplat_frame* frame);
/* densify_and_prune (trainer.cpp:188-275) with the config's thresholds (NULL = defaults) on the
 * accumulated screen statistics; the split offsets come from std::mt19937_64(rng_seed) through
 * std::normal_distribution<double> exactly as in the reference (Trainer::run seeds it with
 * mix64(seed ^ mix64(0x5eed + iteration)), trainer.cpp:370). The planes are reallocated: frames
 * rendered before and device views taken before are invalid afterwards. Gradients, screen
 * statistics and max radii restart at zero (GradientBuffer/DensifyStats::resize); Adam moments
 * of kept Gaussians are carried, new ones start at zero. out may be NULL. */
OSPLAT_API osplat_status osplat_gpu_densify_and_prune(osplat_gpu* ctx, const osplat_config* config, double scene_extent,
                                                      unsigned long long rng_seed, int radius_prune_active,
                                                      osplat_edit_summary* out);
/* reset_opacity (trainer.cpp:277-280): opacity logits clamped to logit(ceiling). */
OSPLAT_API osplat_status osplat_gpu_reset_opacity(osplat_gpu* ctx, double ceiling);
/* Host copy of DensifyStats.max_radius_px (n doubles). */
OSPLAT_API osplat_status osplat_gpu_max_radius(osplat_gpu* ctx, double* max_radius_px);
/* splitmix64 of the trainer's RNG streams (trainer.cpp:300-306). */
OSPLAT_API unsigned long long osplat_mix64(unsigned long long x);

/* ---- optimizer-state sidecar and the training loop ---- */
/* save/load_optimizer_state (dataio.cpp:479-527): the "OSPLADAM" v1 file of the reference
 * (iteration, Adam step, basis count, ten moment arrays as doubles in AdamState layouts). Loading
 * requires a cloud of the same size and basis count; *iteration receives the stored iteration. */
OSPLAT_API osplat_status osplat_gpu_save_state(osplat_gpu* ctx, const char* path, long iteration);
OSPLAT_API osplat_status osplat_gpu_load_state(osplat_gpu* ctx, const char* path, long* iteration);

/* An H x W x 3 double image from host pixels (the Image of image.hpp) — training targets. */
OSPLAT_API osplat_status osplat_image_create(int width, int height, const double* rgb, osplat_image** out);

/* capi.h:58 */
typedef void (*osplat_progress_fn)(void* user, long iteration, double loss, size_t gaussians);
/* osplat_train (capi.cpp:190-234) on the device over an in-memory view set instead of a
 * manifest dataset: views poses (row-major 4x4 world->camera, 16 doubles each) and images
 * (equal sizes); is_test (NULL = all train) selects held-out views (the first one, else the
 * first training view, is rendered for the PSNR of each log line). Trains the context's current
 * cloud from start_iteration (Trainer::resume semantics; 0 = fresh) to config->iterations with
 * Trainer::run's schedule (trainer.cpp:352-392): shuffled views per epoch, SH warm-up, loss,
 * backward, densify/prune/opacity reset, Adam. scene_extent <= 0 uses the reference rule
 * (trainer.cpp:282-298: camera centres, else the cloud's positions). With output_dir set it
 * writes metrics.jsonl, checkpoint_%06ld.ply every checkpoint_interval, final.ply and
 * final.adam like osplat_train; progress (may be NULL) is called on log iterations. */
OSPLAT_API osplat_status osplat_gpu_train(osplat_gpu* ctx, const osplat_config* config, size_t views,
                                          const double* transforms_cw, const osplat_image* const* images,
                                          const uint8_t* is_test, double scene_extent, long start_iteration,
                                          const char* output_dir, osplat_progress_fn progress, void* user);

/* Profiling (bench.py roofline evidence). With timing on, every kernel family is bracketed by a
 * CUDA event pair on the context stream; with count_work on, K3 also writes per-pixel visited
 * list entries so osplat_frame_work can report the algorithmic pair counts. */
#define OSPLAT_KERNEL_COUNT 11
OSPLAT_API osplat_status osplat_gpu_profile(osplat_gpu* ctx, int timing, int count_work);
/* ms[k] / launches[k] for k < OSPLAT_KERNEL_COUNT (synchronizes); reset != 0 clears them. */
OSPLAT_API osplat_status osplat_gpu_profile_read(osplat_gpu* ctx, double* ms, long* launches, int reset);
OSPLAT_API const char* osplat_kernel_name(int id);
/* Work of one frame: forward pairs visited (sum over pixels of list entries evaluated before the
 * T stop), backward pairs (sum of last_contrib), tile instances M. Needs count_work at render. */
OSPLAT_API osplat_status osplat_frame_work(const osplat_frame* frame, uint64_t* fwd_pairs, uint64_t* bwd_pairs,
                                           uint64_t* instances);

/* Kernel launches issued by this library since load (evidence for the benchmark). */
OSPLAT_API long long osplat_gpu_launch_count(void);

#ifdef __cplusplus
}
#endif

#endif /* OSPLAT_B200_H */
