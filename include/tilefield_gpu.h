/*
 * tilefield_gpu.h — C-ABI of the B200-native Snake-NeRF window hot path.
 *
 * This is the drop-in boundary the reference's shared C API would have held
 * (`add_library(tilefield SHARED capi/capi.cpp)`, proj/src/CMakeLists.txt:28-35,
 * hidden visibility; the capi/ and include/ trees are absent upstream).  Every
 * entry point is `extern "C"`, takes plain pointers and sizes, returns an int
 * status (0 = OK) and never lets a C++ exception cross the ABI; the message of
 * the last failure on the calling thread is available from tfg_last_error().
 * A header-only C++ wrapper that rethrows `tilefield::Error` in the reference's
 * style lives in tilefield_gpu.hpp.
 *
 * Device memory is owned by the context; host buffers are caller-owned and are
 * copied (through the context's pinned staging) inside the call.  One context
 * per GPU; calls on a context are ordered on its stream.  There is no CPU
 * fallback: creating a context without an sm_100 device fails.
 *
 * Reference interfaces replaced (file:line under /root/reference/proj/src/):
 *   RationalCamera / project / localize / ray_from_pixel   core/camera.hpp:22-67
 *   crop_for_tile                                          core/camera.hpp:71-72
 *   Roi / TileGrid::build / candidate_tiles                core/tiler.hpp:10-82
 *   intersect_ray_aabb / TileBoxSet::segments             core/geometry.hpp:62-70
 *   FieldConfig                                            core/nn.hpp:14-37
 *   RaySegmentBatch                                        core/ray_batch.hpp:13-49
 *   forward_batch / backward_batch                         core/field.hpp:186-197
 *   adam_step / AdamConfig / LrSchedule                    core/field.hpp:16-48
 *   OccupancyGrid / TileField::update_occupancy            core/field.hpp:55-102
 *   TileField::create / GlobalColorNet::create             core/field.hpp:93,118
 *   save/load_tile_checkpoint (window slide storage tier)  core/field.hpp:206-210
 *   sample_segments / render / color_loss
 *   snake_path / advance / accept_rays / memory_report
 */
#ifndef TILEFIELD_GPU_H
#define TILEFIELD_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(_WIN32)
#define TFG_API
#else
#define TFG_API __attribute__((visibility("default")))
#endif

/* ---- status codes -------------------------------------------------------- */
enum {
    TFG_OK = 0,
    TFG_ERR_INVALID = 1,      /* bad argument / precondition (reference: require) */
    TFG_ERR_CUDA = 2,         /* CUDA runtime failure                              */
    TFG_ERR_NONFINITE = 3,    /* non-finite gradient (field.hpp:45-48)            */
    TFG_ERR_NO_DEVICE = 4,    /* no sm_100 device: there is no CPU fallback        */
    TFG_ERR_STATE = 5         /* call out of order (e.g. step before set_window)   */
};

/* ---- plain data mirrors of the reference types --------------------------- */

/* RationalCamera, core/camera.hpp:22-33 (90 doubles + 2 ints). */
typedef struct tfg_rpc {
    double line_num[20], line_den[20], samp_num[20], samp_den[20];
    double line_off, samp_off, lat_off, long_off, height_off;
    double line_scale, samp_scale, lat_scale, long_scale, height_scale;
    int32_t image_rows, image_cols;
} tfg_rpc;

/* Roi, core/tiler.hpp:10-19. */
typedef struct tfg_roi {
    double easting_min, easting_max;
    double northing_min, northing_max;
    double z_min, z_max;
} tfg_roi;

/* FieldConfig, core/nn.hpp:14-37.  The hash-grid geometry is free (n_min,
 * n_max, table_size: a power of two in [2^4, 2^22]); the widths are the
 * tensor-core kernels' tile shapes, and tfg_create rejects any value other
 * than the default for levels (8), features (2), density_hidden (64),
 * embedding (15), color_hidden (64), color_layers (2), view_freqs (4) and
 * occupancy_resolution (32). */
typedef struct tfg_field_config {
    int32_t levels, table_size, features, n_min, n_max;
    int32_t density_hidden, embedding, color_hidden, color_layers, view_freqs;
    float density_max;
    int32_t occupancy_resolution;
    float occupancy_decay, occupancy_threshold;
    int32_t occupancy_interval;
} tfg_field_config;

/* Trainer / sampler knobs: AdamConfig + LrSchedule (field.hpp:16-31), sampler
 * policy, seeds (rng.hpp:8-10).  See DESIGN.md "pins". */
typedef struct tfg_train_config {
    uint64_t seed;               /* run seed: pixel draws, jitter, init, occupancy */
    double samples_per_meter;    /* per-segment interval density     */
    int32_t max_samples_per_ray; /* per-ray cap                */
    double delta_cap;            /* cap of the final delta in meters */
    float background[3];         /* fixed background RGB             */
    int32_t margin_px;           /* crop dilation (default 4)         */
    double lr_field, lr_color;   /* LrSchedule.base per group        */
    double lr_decay_rate;        /* LrSchedule.decay_rate (1 = constant)           */
    uint64_t lr_decay_steps;     /* LrSchedule.decay_steps                         */
    float beta1, beta2, eps;     /* AdamConfig                                     */
    int32_t batch_rays;          /* global batch size B (loss normaliser)          */
} tfg_train_config;

/* Ray-ordered batch export, the layout of RaySegmentBatch (ray_batch.hpp:13-49).
 * Caller allocates: rays: n_rays; offsets: n_rays+1; per-sample arrays: capacity. */
typedef struct tfg_ray_entry {
    double origin[3];
    double direction[3];
    float target[3];
    int32_t image_id;
    int32_t row, col;
} tfg_ray_entry;

typedef struct tfg_batch_view {
    tfg_ray_entry* rays;
    uint32_t* offsets;
    float* t;
    float* delta;
    float* local;      /* 3 per sample */
    uint8_t* slot;
    uint8_t* endpoint;
    uint64_t capacity; /* sample capacity of the per-sample arrays */
} tfg_batch_view;

/* Per-slot tile state in the reference checkpoint layout (field.hpp:85-109):
 * enc tables | dnet params; Adam m and v for each; step counts; occupancy EMA. */
typedef struct tfg_tile_state {
    float* enc;        /* 434,292 floats (HashGridT::tables)          */
    float* dnet;       /* 2,128 floats   (MlpT params, flat)          */
    float* enc_m;
    float* enc_v;
    float* dnet_m;
    float* dnet_v;
    uint64_t enc_step, dnet_step;
    float* occupancy;  /* res^3 EMA values, x fastest (field.hpp:59)  */
} tfg_tile_state;

typedef struct tfg_memory_report {
    uint64_t tile_params, optimizer_moments, occupancy, crops, accept_list, batch_buffers,
        color_net, staging, total_device;
} tfg_memory_report;

typedef struct tfg_ctx tfg_ctx;

/* ---- lifecycle ----------------------------------------------------------- */
TFG_API const char* tfg_last_error(void);
TFG_API int tfg_default_field_config(tfg_field_config* out);
TFG_API int tfg_default_train_config(tfg_train_config* out);

/* Sizes of one tile's parameter groups for a config (HashGridT::param_count,
 * MlpT::param_count; nn.hpp:57-62,197). */
TFG_API int tfg_param_counts(const tfg_field_config* cfg, uint64_t* enc, uint64_t* dnet,
                             uint64_t* color);

/* Creates a context on `device`; `max_rays` bounds the rays of one batch (per
 * rank).  All device buffers are allocated here (constant HBM footprint). */
TFG_API int tfg_create(const tfg_field_config* fcfg, const tfg_train_config* tcfg, int device,
                       int max_rays, tfg_ctx** out);
TFG_API int tfg_destroy(tfg_ctx* ctx);
/* Orders all subsequent work of the context on `stream` (a cudaStream_t). */
TFG_API int tfg_set_stream(tfg_ctx* ctx, void* stream);

/* ---- scene: cameras, images, grid ---------------------------------------- */
/* Cameras (n_views) and full 8-bit RGB views (rows*cols*3 each, row-major from
 * the top row, image.hpp:10-18).  Images stay in (pinned) host memory; only the
 * window's crops are copied to HBM. */
TFG_API int tfg_set_scene(tfg_ctx* ctx, const tfg_rpc* cams, int n_views,
                          const uint8_t* const* images, const tfg_roi* roi, int grid_rows,
                          int grid_cols);

/* ---- window slide (out-of-core) ------------------------- */
/* Places the 2x2 window with its SW tile at (pos_row, pos_col): evicts the
 * tiles leaving the window to their host records, loads the entering tiles
 * (fresh TileField::create when never trained), stages the window crops and
 * builds the accepted-ray list.  Copies run on a side stream. */
TFG_API int tfg_set_window(tfg_ctx* ctx, int pos_row, int pos_col);
/* Loaded tile of each slot (row, col); slot order is the segment tie order. */
TFG_API int tfg_window_tiles(tfg_ctx* ctx, int32_t* rows4, int32_t* cols4);
/* Snake path: writes (H-1)(W-1) positions as row,col pairs. */
TFG_API int tfg_snake_path(int grid_rows, int grid_cols, int32_t* out_pairs, int* n_out);
/* Prefetch of the next window position's tiles + crops on the side stream. */
TFG_API int tfg_prefetch_window(tfg_ctx* ctx, int pos_row, int pos_col);

/* The accept pass solves every candidate pixel's ray once per window position
 * into a per-window pixel memo (sized by the window's crop union, so HBM is
 * O(1) in the grid size); pixels the previous position already solved are
 * copied from its memo instead of re-solved.  The ray draw reads the memo.
 *
 * Accepted-ray list of the current window: packed
 * (view << 40) | (row << 20) | col, enumerated view, row, col ascending. */
TFG_API int tfg_accept_count(tfg_ctx* ctx, uint64_t* n);
TFG_API int tfg_accept_export(tfg_ctx* ctx, uint64_t* out, uint64_t capacity);

/* ---- one training iteration --------------------------------- */
/* Draws rays [ray_begin, ray_begin + n_rays) of iteration `iter` from the
 * global counter-RNG stream, samples, renders, backpropagates.  Gradients are
 * left in the context's flat gradient buffer (for an allreduce) ... */
TFG_API int tfg_forward_backward(tfg_ctx* ctx, uint64_t iter, uint64_t ray_begin, int n_rays);
/* ... then the fused Adam step over the window's 9 groups plus the periodic
 * occupancy update.  Non-finite gradients raise TFG_ERR_NONFINITE (group named
 * in tfg_last_error) at the next status read. */
TFG_API int tfg_optimizer_step(tfg_ctx* ctx, uint64_t iter);
/* Convenience: forward_backward + optimizer_step + loss readback. */
TFG_API int tfg_train_step(tfg_ctx* ctx, uint64_t iter, uint64_t ray_begin, int n_rays,
                           float* loss_out);
/* Device pointer + float count of the flat gradient buffer (allreduce target). */
TFG_API int tfg_grad_buffer(tfg_ctx* ctx, void** dptr, uint64_t* count);
/* Loss of the last forward_backward (sum over this rank's rays, already
 * divided by 3*B); copies to host and synchronises. */
TFG_API int tfg_read_loss(tfg_ctx* ctx, float* loss_out);

/* Pipelined form of tfg_read_loss: tfg_loss_request enqueues an asynchronous
 * snapshot of the loss / status of the work enqueued so far (at most 4
 * outstanding); tfg_loss_poll waits for the oldest one and reports it exactly
 * as tfg_read_loss does (errors, the non-finite rollback).  A training loop
 * requests after step i and polls after enqueueing step i+1, so the host never
 * waits for the stream to drain. */
TFG_API int tfg_loss_request(tfg_ctx* ctx);
TFG_API int tfg_loss_poll(tfg_ctx* ctx, float* loss_out);

/* ---- multi-GPU: ray-sharded data parallelism (SURVEY.md §8b tfg_comm_init,
 * §8e).  One context per GPU; every rank holds the same window and draws rays
 * [rank * B, (rank + 1) * B) of each iteration, with batch_rays = B * nranks
 * in the train config, so the summed gradient is the global-batch gradient.
 * NCCL is loaded at run time (libnccl.so.2).  Usage per iteration:
 *   tfg_forward_backward; tfg_allreduce_grads; tfg_optimizer_step.
 * Rank 0 creates the id and the host distributes its 128 bytes. */
#define TFG_COMM_ID_BYTES 128
TFG_API int tfg_comm_unique_id(uint8_t* id /* TFG_COMM_ID_BYTES */);
TFG_API int tfg_comm_init(tfg_ctx* ctx, const uint8_t* id, int rank, int nranks);
/* In-place sum of the flat gradient buffer over the ranks, on the context's
 * stream (ordered between the backward and the optimizer step). */
TFG_API int tfg_allreduce_grads(tfg_ctx* ctx);
/* Releases the communicator (tfg_destroy does too). */
TFG_API int tfg_comm_destroy(tfg_ctx* ctx);

/* ---- sub-steps exposed for parity (reference-facing operator surface) ---- */
/* sample_segments over the current window: builds the device batch. */
TFG_API int tfg_sample(tfg_ctx* ctx, uint64_t iter, uint64_t ray_begin, int n_rays, int jitter,
                       uint64_t* n_samples);
/* Builds a batch from caller-given pixels (view,row,col triplets) with jitter
 * off — the render / evaluation path. */
TFG_API int tfg_sample_pixels(tfg_ctx* ctx, const int32_t* pixels, int n_rays,
                              uint64_t* n_samples);
TFG_API int tfg_batch_export(tfg_ctx* ctx, tfg_batch_view* out);
/* A caller-built RaySegmentBatch becomes the current batch (replaces the batch
 * argument of forward_batch / backward_batch, field.hpp:186-197; layout
 * ray_batch.hpp:13-49): rays[n_rays], offsets[n_rays+1] (offsets[0] = 0),
 * per-sample t, delta, local (3), slot, endpoint; capacity is ignored.  Slots
 * index the loaded tiles (set_window, or set_slot_params without a window);
 * each ray's samples must be at most one run per slot. */
TFG_API int tfg_batch_import(tfg_ctx* ctx, const tfg_batch_view* batch, int n_rays);
/* FieldParamView / ColorParamView (field.hpp:130-144): caller-owned parameters
 * into a slot (enc 434,292 + dnet 2,128 floats; NULL keeps) or the colour net
 * (6,915).  With no window set, slots 0..3 are bound detached (forward and
 * backward only). */
TFG_API int tfg_set_slot_params(tfg_ctx* ctx, int slot, const float* enc, const float* dnet);
TFG_API int tfg_set_color_params(tfg_ctx* ctx, const float* params);
/* Caller-given per-sample sigma and rgb (ray order) as the batch's field
 * outputs: tfg_composite then renders exactly these (render alone, SPEC.md:
 * 361-384). */
TFG_API int tfg_set_field_outputs(tfg_ctx* ctx, const float* sigma, const float* rgb);
/* backward_batch (field.hpp:193-197) from caller-given d_sigma / d_rgb (ray
 * order, gradients w.r.t. the outputs of the preceding tfg_field_forward) into
 * the flat gradient buffer (zeroed first; read with tfg_get_grads). */
TFG_API int tfg_field_backward_from(tfg_ctx* ctx, const float* d_sigma, const float* d_rgb);
/* adam_step (field.hpp:45-48) over caller spans, host or device memory:
 * AdamState = (m, v, *step), LrSchedule = (lr_base, lr_decay_rate,
 * lr_decay_steps), AdamConfig = (beta1, beta2, eps).  Non-finite gradients:
 * TFG_ERR_NONFINITE naming `group`, nothing updated, *step unchanged; else
 * *step += 1.  Bit-identical to the reference formula. */
TFG_API int tfg_adam_step(tfg_ctx* ctx, float* params, const float* grads, float* m, float* v, uint64_t n,
                          uint64_t* step, double lr_base, double lr_decay_rate, uint64_t lr_decay_steps,
                          float beta1, float beta2, float eps, const char* group);
/* forward_batch: per-sample sigma and rgb in ray order (n_samples, 3*n_samples). */
TFG_API int tfg_field_forward(tfg_ctx* ctx, float* sigma, float* rgb);
/* render + color_loss + render backward: per-ray rgb(3)/depth/opacity, and the
 * per-sample d_sigma / d_rgb in ray order (any output may be NULL). */
TFG_API int tfg_composite(tfg_ctx* ctx, float* ray_rgb, float* ray_depth, float* ray_opacity,
                          float* d_sigma, float* d_rgb, float* loss);
/* backward_batch of the tfg_composite gradients into the flat gradient buffer
 * (zeroed first); needs tfg_field_forward of this batch first. */
TFG_API int tfg_field_backward(tfg_ctx* ctx);

/* ---- parameter / state access -------------------------------------------- */
TFG_API int tfg_get_tile_state(tfg_ctx* ctx, int slot, tfg_tile_state* out);
TFG_API int tfg_set_tile_state(tfg_ctx* ctx, int slot, const tfg_tile_state* in);
TFG_API int tfg_get_color(tfg_ctx* ctx, float* params, float* m, float* v, uint64_t* step);
TFG_API int tfg_set_color(tfg_ctx* ctx, const float* params, const float* m, const float* v,
                          uint64_t step);
/* Gradients of the last backward: per slot enc (434,292) + dnet (2,128), colour. */
TFG_API int tfg_get_grads(tfg_ctx* ctx, int slot, float* enc, float* dnet, float* color);
TFG_API int tfg_update_occupancy(tfg_ctx* ctx);
TFG_API int tfg_get_memory_report(tfg_ctx* ctx, tfg_memory_report* out);

/* ---- crop cache (build_crop_cache; §8(f) row 3) --------
 * Per-(view, tile) crop rasters of the scene (crop_for_tile, camera.cpp:
 * 126-146, with TrainConfig.margin_px) and an index, little-endian:
 *   "TFCROP01" | u32 version (1) | u32 n_views | u32 grid_rows | u32 grid_cols
 *   | i32 margin_px | u32 0 | u64 n_entries | u64 data_offset
 *   | n_entries x { i32 view, tile_row, tile_col, r0, r1, c0, c1, 0;
 *                   u64 offset, u64 bytes }      (view-major, then row, col)
 *   | u8 RGB crops, row-major, at data_offset + offset.
 * Empty crops have r0 = r1 = c0 = c1 = 0 and 0 bytes.  load_crop_cache
 * rejects a cache whose grid, margin or any rect differs from this scene's,
 * then fills the pinned host images (after set_scene, which may take NULL
 * images) so that training reads only cached crops. */
TFG_API int tfg_build_crop_cache(tfg_ctx* ctx, const char* path, uint64_t* total_crop_bytes);
TFG_API int tfg_load_crop_cache(tfg_ctx* ctx, const char* path);
TFG_API int tfg_crop_rect(tfg_ctx* ctx, int view, int tile_row, int tile_col, int32_t* r0r1c0c1);

/* ---- evaluation (evalio; §8(f) row 2) --------------------
 * Host buffers in, computed on the context's GPU (FP64 sums).
 *   psnr: a, b hold n values in [0,1]; 10 log10(1/MSE), capped at 99 dB.
 *   ssim: rows x cols x 3 RGB; grey = channel mean, 11x11 Gaussian sigma 1.5,
 *         K1 0.01, K2 0.03, L 1; mean over the valid windows.
 *   depth_mae: mean |d1 - d2| over mask != 0 (mask may be NULL = all).
 *   edge_band_mask: 1 within +-band_px of the projected tile edges (the grid
 *         boundary lines at z_min and z_max) in view `cam`, else 0.
 *   render_view: full-frame render of `cam` (row-major, every pixel) through
 *         the render path (render_setup first). */
TFG_API int tfg_psnr(tfg_ctx* ctx, const float* a, const float* b, uint64_t n, double* db);
TFG_API int tfg_ssim(tfg_ctx* ctx, const float* a, const float* b, int rows, int cols, double* ssim);
TFG_API int tfg_depth_mae(tfg_ctx* ctx, const float* d1, const float* d2, const uint8_t* mask, uint64_t n,
                          double* mae);
TFG_API int tfg_edge_band_mask(tfg_ctx* ctx, const tfg_rpc* cam, int band_px, uint8_t* mask);
TFG_API int tfg_render_view(tfg_ctx* ctx, const tfg_rpc* cam, float* rgb, float* depth, float* opacity);

/* ---- checkpoints (save/load_tile_checkpoint, save/load_color_checkpoint,
 * field.hpp:202-210) ---------------------------------------
 * Versioned little-endian binary: "TFCKPT01" | u32 version (1) | u32 kind
 * (1 tile, 2 colour net) | tfg_field_config | i32 row, col | u64 n_params,
 * n_occupancy | u64 step(s) | f32 params | f32 m | f32 v | f32 occupancy.
 * Round trips are bit-exact; a mismatching FieldConfig is rejected. */
TFG_API int tfg_save_tile_checkpoint(const char* path, const tfg_field_config* cfg, int row, int col,
                                     const tfg_tile_state* st);
TFG_API int tfg_load_tile_checkpoint(const char* path, const tfg_field_config* cfg, int* row, int* col,
                                     tfg_tile_state* st);
TFG_API int tfg_save_color_checkpoint(const char* path, const tfg_field_config* cfg, const float* params,
                                      const float* m, const float* v, uint64_t step);
TFG_API int tfg_load_color_checkpoint(const char* path, const tfg_field_config* cfg, float* params,
                                      float* m, float* v, uint64_t* step);
/* Whole run state: every tile ever loaded (tiles/r{R}_c{C}.ckpt, from the
 * window slots or the host records) + color_net.ckpt under `dir` (which must
 * exist, with a tiles/ subdirectory); load restores it into a context after
 * set_scene (before set_window). */
TFG_API int tfg_save_run(tfg_ctx* ctx, const char* dir);
TFG_API int tfg_load_run(tfg_ctx* ctx, const char* dir);

/* ---- render path (cmd_render; config 4) --------------------- */
/* Loads up to `n_tiles` tiles (params only) for forward-only rendering over
 * an ROI sub-grid; tile_state entries need enc, dnet, occupancy. */
TFG_API int tfg_render_setup(tfg_ctx* ctx, const int32_t* rows, const int32_t* cols, int n_tiles,
                             const tfg_tile_state* states, const float* color_params);
/* Renders caller-given rays of camera `cam` (pixels as row,col pairs):
 * per-ray rgb(3), depth, opacity to host. */
TFG_API int tfg_render_pixels(tfg_ctx* ctx, const tfg_rpc* cam, const int32_t* pixels,
                              int n_rays, float* rgb, float* depth, float* opacity);

/* ---- timing helpers (kernel share inside the timed region) --------------- */
/* Accumulated device milliseconds and launch counts per kernel family since
 * the last reset (CUDA events on the context stream; enabled by flag). */
TFG_API int tfg_profile_enable(tfg_ctx* ctx, int on);
TFG_API int tfg_profile_read(tfg_ctx* ctx, const char** names, double* ms, uint64_t* launches,
                             int capacity, int* n_out);
TFG_API int tfg_kernel_launch_count(tfg_ctx* ctx, uint64_t* launches);
/* Rays and samples of the last batch (synchronises). */
TFG_API int tfg_last_batch(tfg_ctx* ctx, int* n_rays, uint64_t* n_samples);
/* TileField::create (field.hpp:93) on the host into caller buffers. */
TFG_API int tfg_tile_init(const tfg_field_config* cfg, uint64_t seed, int row, int col,
                          tfg_tile_state* out);
/* Host<->device bytes copied by the context (window slides, crops, status). */
TFG_API int tfg_copy_bytes(tfg_ctx* ctx, uint64_t* h2d, uint64_t* d2h);

#ifdef __cplusplus
}
#endif

#endif /* TILEFIELD_GPU_H */
