// tilefield_gpu_field.hpp — header-only drop-in of the reference's batch
// operators with their field.hpp signatures, over the C-ABI:
//
//   forward_batch<S>   (field.hpp:185-188)  RaySegmentBatch + FieldParamView[]
//                                           + ColorParamView -> ws.sigma, ws.rgb
//   backward_batch<S>  (field.hpp:190-197)  + d_sigma, d_rgb -> BatchGrads
//   adam_step          (field.hpp:45-48)    params, grads, AdamState, LrSchedule,
//                                           AdamConfig, group
//
// The calls run on a per-thread default context (set_default_context): the
// caller's spans are copied into its HBM, the sm_100a kernels run, and the
// results are copied back, so a reference trainer keeps its own data
// structures.  S must be float (the GPU path is fp32/bf16; the reference's
// float64 instantiation is its finite-difference oracle).  Errors throw
// tilefield::Error with the reference's messages (non-finite gradients name
// the parameter group).
//
// Types: built inside the reference tree (TILEFIELD_GPU_REFERENCE_TYPES
// defined, core/ on the include path) the functions take the reference's own
// RaySegmentBatch / FieldParamView / ... (Eigen vectors are indexed with []).
// Standalone, this header declares layout-compatible mirrors of those types
// in namespace tilefield (same member names), used by the repo's tests.
#pragma once

#include <cmath>
#include <cstdint>
#include <span>
#include <string>
#include <type_traits>
#include <vector>

#include "tilefield_gpu.hpp"

#ifdef TILEFIELD_GPU_REFERENCE_TYPES
#include "core/field.hpp"
#else
namespace tilefield {

// ---- mirrors of the reference types (common.hpp, ray_batch.hpp, field.hpp)
struct PixelRc {
    int row = 0, col = 0;
};
using FieldConfig = tfg_field_config;

struct RaySegmentBatch {  // ray_batch.hpp:13-49
    struct RayEntry {
        double origin[3] = {0, 0, 0};
        double direction[3] = {0, 0, 0};
        float target[3] = {0, 0, 0};
        int image_id = -1;
        PixelRc pixel;
    };
    std::vector<RayEntry> rays;
    std::vector<uint32_t> offsets;  // rays.size() + 1
    std::vector<float> t, delta, local;
    std::vector<uint8_t> slot, endpoint;
    size_t ray_count() const { return rays.size(); }
    size_t sample_count() const { return t.size(); }
};

template <typename S>
struct FieldParamView {  // field.hpp:130-137 (topology pointers unused here)
    const FieldConfig* cfg = nullptr;
    const void* grid = nullptr;
    const void* dnet = nullptr;
    const S* enc_tables = nullptr;
    const S* dnet_params = nullptr;
};

template <typename S>
struct ColorParamView {  // field.hpp:139-144
    const FieldConfig* cfg = nullptr;
    const void* net = nullptr;
    const S* params = nullptr;
};

template <typename S>
struct ForwardWorkspace {  // field.hpp:147-165
    std::vector<S> view_enc, dnet_acts, cnet_acts, sigma_raw, sigma, rgb;
};

template <typename S>
struct FieldGrads {
    std::vector<S> enc, dnet;
};

template <typename S>
struct BatchGrads {  // field.hpp:170-183
    std::vector<FieldGrads<S>> tiles;
    std::vector<S> color;
};

struct AdamConfig {  // field.hpp:16-20
    float beta1 = 0.9f, beta2 = 0.99f, eps = 1e-15f;
};
struct LrSchedule {  // field.hpp:22-31
    double base = 1e-2, decay_rate = 1.0;
    uint64_t decay_steps = 1000;
};
struct AdamState {  // field.hpp:33-43
    std::vector<float> m, v;
    uint64_t step = 0;
};

}  // namespace tilefield
#endif

namespace tilefield {
namespace gpu {

inline Context*& default_context_slot() {
    thread_local Context* ctx = nullptr;
    return ctx;
}
// The context the drop-in operators run on (one per GPU / host thread).
inline void set_default_context(Context* ctx) { default_context_slot() = ctx; }
inline Context& default_context() {
    Context* c = default_context_slot();
    if (!c) throw Error("tilefield::gpu: set_default_context() before forward_batch/backward_batch/adam_step");
    return *c;
}

namespace detail {
template <class FP, class CP>
void load_params(Context& ctx, std::span<const FP> tiles, const CP& color) {
    for (size_t k = 0; k < tiles.size(); ++k)
        check(tfg_set_slot_params(ctx.raw(), int(k), tiles[k].enc_tables, tiles[k].dnet_params));
    check(tfg_set_color_params(ctx.raw(), color.params));
}

template <class Batch>
void import_batch(Context& ctx, const Batch& batch) {
    const size_t n = batch.rays.size();
    std::vector<tfg_ray_entry> rays(n);
    for (size_t i = 0; i < n; ++i) {
        const auto& r = batch.rays[i];
        for (int q = 0; q < 3; ++q) {
            rays[i].origin[q] = r.origin[q];
            rays[i].direction[q] = r.direction[q];
            rays[i].target[q] = r.target[q];
        }
        rays[i].image_id = r.image_id;
        rays[i].row = r.pixel.row;
        rays[i].col = r.pixel.col;
    }
    tfg_batch_view v{};
    v.rays = rays.data();
    v.offsets = const_cast<uint32_t*>(batch.offsets.data());
    v.t = const_cast<float*>(batch.t.data());
    v.delta = const_cast<float*>(batch.delta.data());
    v.local = const_cast<float*>(batch.local.data());
    v.slot = const_cast<uint8_t*>(batch.slot.data());
    v.endpoint = const_cast<uint8_t*>(batch.endpoint.data());
    v.capacity = batch.t.size();
    check(tfg_batch_import(ctx.raw(), &v, int(n)));
}

inline void require_finite(const std::vector<float>& g, const std::string& group) {
    for (float x : g)
        if (!std::isfinite(x)) throw Error("backward_batch: non-finite gradient in group " + group);
}
}  // namespace detail

// forward_batch (field.hpp:185-188): per-sample sigma and rgb into ws.  The
// GPU keeps the activations it needs for the backward in HBM, so ws's
// activation arrays are left empty.  `workers` is accepted and ignored.
template <typename S>
void forward_batch(const RaySegmentBatch& batch, std::span<const FieldParamView<S>> tiles,
                   const ColorParamView<S>& color, ForwardWorkspace<S>& ws, int workers) {
    static_assert(std::is_same_v<S, float>, "the GPU path computes in fp32 (bf16 tensor-core operands)");
    (void)workers;
    Context& ctx = default_context();
    detail::load_params(ctx, tiles, color);
    detail::import_batch(ctx, batch);
    const size_t n = batch.t.size();
    ws.sigma.resize(n);
    ws.rgb.resize(3 * n);
    check(tfg_field_forward(ctx.raw(), ws.sigma.data(), ws.rgb.data()));
}

// backward_batch (field.hpp:190-197): parameter gradients from d_sigma /
// d_rgb of the preceding forward_batch of the same batch on this thread's
// context.  Gradients are written (not accumulated) into `grads`, sized like
// the parameter groups; non-finite gradients throw naming the group.
template <typename S>
void backward_batch(const RaySegmentBatch& batch, std::span<const FieldParamView<S>> tiles,
                    const ColorParamView<S>& color, const ForwardWorkspace<S>& ws, std::span<const S> d_sigma,
                    std::span<const S> d_rgb, BatchGrads<S>& grads, int workers) {
    static_assert(std::is_same_v<S, float>, "the GPU path computes in fp32 (bf16 tensor-core operands)");
    (void)color;
    (void)workers;
    if (ws.sigma.size() != batch.t.size() || d_sigma.size() != batch.t.size() || d_rgb.size() != 3 * batch.t.size())
        throw Error("backward_batch: workspace / gradient sizes do not match the batch");
    Context& ctx = default_context();
    check(tfg_field_backward_from(ctx.raw(), d_sigma.data(), d_rgb.data()));
    uint64_t enc = 0, dnet = 0, col = 0;
    tfg_field_config fc{};
    check(tfg_default_field_config(&fc));
    check(tfg_param_counts(&fc, &enc, &dnet, &col));
    grads.tiles.resize(tiles.size());
    grads.color.assign(col, 0.f);
    for (size_t k = 0; k < tiles.size(); ++k) {
        grads.tiles[k].enc.assign(enc, 0.f);
        grads.tiles[k].dnet.assign(dnet, 0.f);
        check(tfg_get_grads(ctx.raw(), int(k), grads.tiles[k].enc.data(), grads.tiles[k].dnet.data(),
                            k == 0 ? grads.color.data() : nullptr));
    }
    for (size_t k = 0; k < tiles.size(); ++k) {
        detail::require_finite(grads.tiles[k].enc, "slot" + std::to_string(k) + ".enc");
        detail::require_finite(grads.tiles[k].dnet, "slot" + std::to_string(k) + ".dnet");
    }
    detail::require_finite(grads.color, "color");
}

// adam_step (field.hpp:45-48): one Adam update of `params` (host span) on
// the GPU, bit-identical to the reference formula; throws on non-finite
// gradients naming `group`, leaving params and state untouched.
inline void adam_step(std::span<float> params, std::span<const float> grads, AdamState& state,
                      const LrSchedule& schedule, const AdamConfig& cfg, const std::string& group) {
    if (grads.size() != params.size() || state.m.size() != params.size() || state.v.size() != params.size())
        throw Error("adam_step: size mismatch in group " + group);
    Context& ctx = default_context();
    uint64_t step = state.step;
    check(tfg_adam_step(ctx.raw(), params.data(), grads.data(), state.m.data(), state.v.data(), params.size(), &step,
                        schedule.base, schedule.decay_rate, schedule.decay_steps, cfg.beta1, cfg.beta2, cfg.eps,
                        group.c_str()));
    state.step = step;
}

}  // namespace gpu
}  // namespace tilefield
