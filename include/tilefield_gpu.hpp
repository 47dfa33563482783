// tilefield_gpu.hpp — header-only C++ mirror of the reference's tile-grid /
// window / sampler / trainer API over the C-ABI (tilefield_gpu.h).
//
// Errors surface as tilefield::Error (core/common.hpp:27-30 of the reference)
// with the library's message, so reference-side callers keep their error
// handling.  The reference types RationalCamera (camera.hpp:22-33), Roi
// (tiler.hpp:10-19) and FieldConfig (nn.hpp:14-37) map 1:1 onto tfg_rpc,
// tfg_roi and tfg_field_config; see INTEGRATION.md for the adapter that
// implements forward_batch / backward_batch / adam_step on top of this.
#pragma once

#include <array>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "tilefield_gpu.h"

namespace tilefield {

#ifndef TILEFIELD_ERROR_DEFINED
#define TILEFIELD_ERROR_DEFINED
class Error : public std::runtime_error {
public:
    explicit Error(const std::string& msg) : std::runtime_error(msg) {}
};
#endif

namespace gpu {

inline void check(int rc) {
    if (rc != TFG_OK) throw Error(tfg_last_error());
}

// One GPU's window trainer (a tfg_ctx): owns HBM state of the 2x2 window.
class Context {
public:
    Context(const tfg_field_config& f, const tfg_train_config& t, int device, int max_rays) {
        check(tfg_create(&f, &t, device, max_rays, &c_));
    }
    ~Context() { tfg_destroy(c_); }
    Context(const Context&) = delete;
    Context& operator=(const Context&) = delete;

    void set_stream(void* stream) { check(tfg_set_stream(c_, stream)); }
    void set_scene(const std::vector<tfg_rpc>& cams, const std::vector<const uint8_t*>& images,
                   const tfg_roi& roi, int rows, int cols) {
        check(tfg_set_scene(c_, cams.data(), int(cams.size()), images.data(), &roi, rows, cols));
    }

    // scheduler: snake_path / advance
    static std::vector<std::pair<int, int>> snake_path(int H, int W) {
        int n = 0;
        check(tfg_snake_path(H, W, nullptr, &n));
        std::vector<int32_t> p(2 * n);
        check(tfg_snake_path(H, W, p.data(), &n));
        std::vector<std::pair<int, int>> out;
        for (int k = 0; k < n; ++k) out.push_back({p[2 * k], p[2 * k + 1]});
        return out;
    }
    void advance(int pos_row, int pos_col) { check(tfg_set_window(c_, pos_row, pos_col)); }
    uint64_t accepted_rays() const {
        uint64_t n = 0;
        check(tfg_accept_count(c_, &n));
        return n;
    }

    // one trainer iteration; loss = color_loss
    float train_step(uint64_t iter, uint64_t ray_begin, int n_rays) {
        float loss = 0.f;
        check(tfg_train_step(c_, iter, ray_begin, n_rays, &loss));
        return loss;
    }
    // split form for data parallelism: fwd/bwd, allreduce(grad_buffer()), step
    void forward_backward(uint64_t iter, uint64_t ray_begin, int n_rays) {
        check(tfg_forward_backward(c_, iter, ray_begin, n_rays));
    }
    std::pair<float*, uint64_t> grad_buffer() {
        void* p = nullptr;
        uint64_t n = 0;
        check(tfg_grad_buffer(c_, &p, &n));
        return {static_cast<float*>(p), n};
    }
    void optimizer_step(uint64_t iter) { check(tfg_optimizer_step(c_, iter)); }
    // the library's own NCCL communicator: rank 0 calls comm_unique_id() and
    // the host distributes the 128 bytes; then per iteration
    // forward_backward, allreduce_grads, optimizer_step
    static std::array<uint8_t, TFG_COMM_ID_BYTES> comm_unique_id() {
        std::array<uint8_t, TFG_COMM_ID_BYTES> id{};
        check(tfg_comm_unique_id(id.data()));
        return id;
    }
    void comm_init(const std::array<uint8_t, TFG_COMM_ID_BYTES>& id, int rank, int nranks) {
        check(tfg_comm_init(c_, id.data(), rank, nranks));
    }
    void allreduce_grads() { check(tfg_allreduce_grads(c_)); }
    float read_loss() {
        float l = 0.f;
        check(tfg_read_loss(c_, &l));
        return l;
    }
    // pipelined: request after step i, poll after enqueueing step i+1
    void request_loss() { check(tfg_loss_request(c_)); }
    float poll_loss() {
        float l = 0.f;
        check(tfg_loss_poll(c_, &l));
        return l;
    }

    // reference-facing operator surface (RaySegmentBatch, forward_batch, render)
    uint64_t sample_segments(uint64_t iter, uint64_t ray_begin, int n_rays, bool jitter) {
        uint64_t n = 0;
        check(tfg_sample(c_, iter, ray_begin, n_rays, jitter ? 1 : 0, &n));
        return n;
    }
    void export_batch(tfg_batch_view* out) { check(tfg_batch_export(c_, out)); }
    void forward_batch(float* sigma, float* rgb) { check(tfg_field_forward(c_, sigma, rgb)); }
    float render_and_loss(float* rgb, float* depth, float* opacity, float* d_sigma, float* d_rgb) {
        float loss = 0.f;
        check(tfg_composite(c_, rgb, depth, opacity, d_sigma, d_rgb, &loss));
        return loss;
    }
    void backward_batch() { check(tfg_field_backward(c_)); }
    // caller-owned data (the reference operators' arguments; the field.hpp
    // signatures themselves are in tilefield_gpu_field.hpp)
    void import_batch(const tfg_batch_view& batch, int n_rays) { check(tfg_batch_import(c_, &batch, n_rays)); }
    void set_slot_params(int slot, const float* enc, const float* dnet) {
        check(tfg_set_slot_params(c_, slot, enc, dnet));
    }
    void set_color_params(const float* params) { check(tfg_set_color_params(c_, params)); }
    void set_field_outputs(const float* sigma, const float* rgb) { check(tfg_set_field_outputs(c_, sigma, rgb)); }
    void backward_batch_from(const float* d_sigma, const float* d_rgb) {
        check(tfg_field_backward_from(c_, d_sigma, d_rgb));
    }
    void grads(int slot, float* enc, float* dnet, float* color) { check(tfg_get_grads(c_, slot, enc, dnet, color)); }
    void tile_state(int slot, tfg_tile_state* out) { check(tfg_get_tile_state(c_, slot, out)); }
    void set_tile_state(int slot, const tfg_tile_state& in) { check(tfg_set_tile_state(c_, slot, &in)); }
    tfg_memory_report memory_report() {
        tfg_memory_report r{};
        check(tfg_get_memory_report(c_, &r));
        return r;
    }

    // render + evaluation (cmd_render, evalio)
    void render_setup(const int32_t* rows, const int32_t* cols, int n, const tfg_tile_state* states,
                      const float* color_params) {
        check(tfg_render_setup(c_, rows, cols, n, states, color_params));
    }
    void render_view(const tfg_rpc& cam, float* rgb, float* depth, float* opacity) {
        check(tfg_render_view(c_, &cam, rgb, depth, opacity));
    }
    double psnr(const float* a, const float* b, uint64_t n) {
        double v = 0.0;
        check(tfg_psnr(c_, a, b, n, &v));
        return v;
    }
    double ssim(const float* a, const float* b, int rows, int cols) {
        double v = 0.0;
        check(tfg_ssim(c_, a, b, rows, cols, &v));
        return v;
    }
    double depth_mae(const float* d1, const float* d2, const uint8_t* mask, uint64_t n) {
        double v = 0.0;
        check(tfg_depth_mae(c_, d1, d2, mask, n, &v));
        return v;
    }
    void edge_band_mask(const tfg_rpc& cam, int band_px, uint8_t* mask) {
        check(tfg_edge_band_mask(c_, &cam, band_px, mask));
    }

    // persistence (checkpoints, run resume, crop cache)
    void save_run(const std::string& dir) { check(tfg_save_run(c_, dir.c_str())); }
    void load_run(const std::string& dir) { check(tfg_load_run(c_, dir.c_str())); }
    uint64_t build_crop_cache(const std::string& path) {
        uint64_t n = 0;
        check(tfg_build_crop_cache(c_, path.c_str(), &n));
        return n;
    }
    void load_crop_cache(const std::string& path) { check(tfg_load_crop_cache(c_, path.c_str())); }

    tfg_ctx* raw() { return c_; }

private:
    tfg_ctx* c_ = nullptr;
};

} // namespace gpu
} // namespace tilefield
