/*
 * tf_oracle.h — TEST INFRASTRUCTURE ONLY (the parity checker, never the product).
 *
 * CPU restatement of the Snake-NeRF window hot path of the reference
 * (/root/reference/proj/src/core, SPEC.md).  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference leg may load this library.
 *
 * Pinning: the restated pieces that exist upstream (rng, camera, geometry,
 * tiler, nn) are checked bit-for-bit against the reference sources compiled
 * verbatim into oracle/_ref/libtfref.so (tests/test_oracle_vs_ref.py).  The
 * pieces that are declared but absent upstream (field.cpp, sampling.cpp,
 * renderer.cpp, scheduler.cpp, trainer.cpp) are restated from SPEC.md and pinned
 * by the SPEC known-answer examples (tests/test_oracle_kat.py); everything the
 * SPEC leaves open is pinned in DESIGN.md §"Pins" and here.
 */
#ifndef TF_ORACLE_H
#define TF_ORACLE_H

#include "../include/tilefield_gpu.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct tfo_session tfo_session;

const char* tfo_last_error(void);

/* ---- primitives (status 0 = ok, 1 = reference would throw) --------------- */
int tfo_project(const tfg_rpc* cam, const double* xyz, double* rc);
int tfo_localize(const tfg_rpc* cam, const double* px, double height, double* xy, double* resid,
                 int* iters);
int tfo_ray_from_pixel(const tfg_rpc* cam, int row, int col, double z_min, double z_max,
                       double* origin, double* dir);
int tfo_intersect(const double* o, const double* d, const double* box6, double* t0, double* t1);
int tfo_segments(const double* o, const double* d, const double* boxes6, int n, int* slot,
                 double* tn, double* tf);
int tfo_crop_for_tile(const tfg_rpc* cam, const double* box6, int margin, int* rect4);
int tfo_grid_edges(const tfg_roi* roi, int rows, int cols, double* east, double* north);
int tfo_candidate_tiles(const tfg_roi* roi, int rows, int cols, const double* o, const double* d,
                        int* rc_pairs, int capacity);
int tfo_snake_path(int rows, int cols, int* pairs, int capacity);
int tfo_level_resolution(const tfg_field_config* cfg, int level);
uint64_t tfo_splitmix64(uint64_t x);
uint64_t tfo_hash_combine(uint64_t a, uint64_t b);

/* Samples one ray over given segments (ray_batch.hpp layout).
 * occupancy: per segment slot a res^3 EMA grid (NULL = fully occupied);
 * frames: per slot origin(3)+inv_size(3).  Returns the sample count, or -1 if
 * capacity is exceeded. */
int tfo_sample_ray(const double* o, const double* d, int n_seg, const int* seg_slot,
                   const double* seg_tn, const double* seg_tf, const double* frames6,
                   const float* const* occupancy, int occ_res, float occ_threshold,
                   double samples_per_meter, int max_samples, double z_min, double delta_cap,
                   int jitter, uint64_t ray_key, float* t, float* delta, float* local,
                   uint8_t* slot, uint8_t* endpoint, int capacity);

/* Volume rendering of one ray + its backward for upstream
 * gradient g_rgb.  d_sigma / d_rgb may be NULL. */
void tfo_render_ray(int n, const float* sigma, const float* rgb, const float* t,
                    const float* delta, const float* bg, float* out_rgb, float* out_depth,
                    float* out_opacity, const float* g_rgb, float* d_sigma, float* d_rgb);

/* cmd_render: (row, col) pixels of `cam` over n_tiles boxes
 * (min xyz, max xyz; slot order = tile order), midpoint samples, per-tile
 * fields, render; failed rays give zeros.  Parallel over `workers`. */
int tfo_render_pixels(const tfg_field_config* cfg, const tfg_rpc* cam, double z_min, double z_max,
                      int n_tiles, const double* boxes6, const float* const* enc, const float* const* dnet,
                      const float* const* occupancy, const float* color, double spm, int cap,
                      double dcap, const float* bg, int n_px, const int32_t* px, float* rgb,
                      float* depth, float* opacity, int workers);

/* Adam on one group (field.hpp:45-48).  Returns 1 (and sets
 * the error naming `group`) on non-finite gradients, parameters untouched. */
int tfo_adam_step(float* params, const float* grads, float* m, float* v, uint64_t n,
                  uint64_t* step, double lr_base, double decay_rate, uint64_t decay_steps,
                  float beta1, float beta2, float eps, const char* group);

/* Fresh tile / colour net (TileField::create, GlobalColorNet::create). */
int tfo_tile_create(const tfg_field_config* cfg, int row, int col, uint64_t seed, float* enc,
                    float* dnet, float* occupancy);
int tfo_color_create(const tfg_field_config* cfg, uint64_t seed, float* params);

/* Per-point field query on explicit parameters (query_density/query_color). */
int tfo_query_field(const tfg_field_config* cfg, const float* enc, const float* dnet,
                    const float* color, const float* local3, const float* dir3, float* sigma,
                    float* rgb);

/* color_loss over n rays with batch size `batch`: returns
 * the loss (mean over rays and channels), writes d loss / d rgb if grad. */
double tfo_color_loss(const float* rgb, const float* target, int n, int batch, float* grad);

/* Backward primitives (pinned against nn.hpp:116-157 / 231-245 by the tests):
 * one MLP forward + backward_p (grad accumulates), and n hash lookups +
 * HashGridT::backward (grad accumulates; d_out/grad may be NULL). */
int tfo_mlp_fwd_bwd(const int* widths, int nw, const float* params, const float* x, float* out,
                    const float* d_out, float* grad, float* d_in);
int tfo_hash_lookup_bwd(const tfg_field_config* cfg, const float* tables, int n, const float* p3,
                        float* out, const float* d_out, float* grad);

/* ---- session: the trainer's window state ---------------------------------- */
tfo_session* tfo_create(const tfg_field_config* fcfg, const tfg_train_config* tcfg,
                        const tfg_rpc* cams, int n_views, const uint8_t* const* images,
                        const tfg_roi* roi, int grid_rows, int grid_cols, int workers);
void tfo_destroy(tfo_session* s);
int tfo_set_window(tfo_session* s, int pos_row, int pos_col);
int tfo_window_tiles(tfo_session* s, int* rows4, int* cols4);
int64_t tfo_build_accept(tfo_session* s);
int64_t tfo_accept_export(tfo_session* s, uint64_t* out, uint64_t capacity);
int64_t tfo_sample(tfo_session* s, uint64_t iter, uint64_t ray_begin, int n_rays, int jitter);
int64_t tfo_sample_pixels(tfo_session* s, const int32_t* pixels, int n_rays);
int tfo_batch_export(tfo_session* s, tfg_batch_view* out);
int tfo_forward(tfo_session* s, float* sigma, float* rgb);
int tfo_composite(tfo_session* s, float* ray_rgb, float* ray_depth, float* ray_opacity,
                  float* d_sigma, float* d_rgb, double* loss);
int tfo_backward(tfo_session* s);
int tfo_get_grads(tfo_session* s, int slot, float* enc, float* dnet, float* color);
int tfo_optimizer_step(tfo_session* s, uint64_t iter);
int tfo_train_step(tfo_session* s, uint64_t iter, uint64_t ray_begin, int n_rays, double* loss);
int tfo_get_tile_state(tfo_session* s, int slot, tfg_tile_state* out);
int tfo_set_tile_state(tfo_session* s, int slot, const tfg_tile_state* in);
int tfo_get_color(tfo_session* s, float* params, float* m, float* v, uint64_t* step);
int tfo_set_color(tfo_session* s, const float* params, const float* m, const float* v,
                  uint64_t step);
int tfo_update_occupancy(tfo_session* s);
int tfo_set_workers(tfo_session* s, int workers);
/* float64 shadow of the current batch's loss and (if g_* != NULL) its exact
 * reverse-mode gradient, parameters per loaded slot (the finite-difference
 * oracle). */
double tfo_shadow_loss_grad(tfo_session* s, const double* const* enc, const double* const* dnet,
                            const double* color, double* const* g_enc, double* const* g_dnet,
                            double* g_color);

#ifdef __cplusplus
}
#endif
#endif
