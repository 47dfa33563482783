// tfg_api.cu — the C-ABI (include/tilefield_gpu.h) over the B200 kernels:
// context and HBM layout, scene + crops, the out-of-core window slide
// (scheduler advance) between pinned host records and HBM on a
// side stream, the training-iteration driver and the render path.
// Persistence is in tfg_io.cu, evaluation in tfg_eval.cu (shared internals:
// tfg_internal.h).
//
// HBM layout (allocated once in tfg_create / tfg_set_scene; constant across
// the snake progression):
//   params / grads / m / v : flat [slot0 enc | slot0 dnet | ... | slot3 | colour]
//                            1,752,595 floats each (the allreduce / Adam span)
//   ema / bits             : 4 x 32^3 occupancy EMA + 4 x 4 KB bitfields
//   crops                  : per-view union of the window's 4 tile crops (u8 RGB)
//   accept                 : packed (view, row, col) accepted-ray list
//   batch                  : RayRec per ray, 24-float view encoding per ray,
//                            slot-bucketed SoA samples (local+ray, t+delta,
//                            endpoint, sigma/rgb -> dsigma/drgb)
#include "tfg_internal.h"

namespace tfg {
namespace host {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

// ---------------------------------------------------------------- host-side field init
// TileField::create / GlobalColorNet::create (field.hpp:93,118) with the
// per-tile streams Rng(hash_combine(seed, purpose, row, col)): HashGridT::init
// U(-1e-4, 1e-4) (nn.hpp:194), MlpT::init Xavier-uniform + zero bias (nn.hpp:70-81).
void mlp_init_host(const int* w, int nw, Rng& rng, float* p) {
    size_t k = 0;
    for (int l = 0; l + 1 < nw; ++l) {
        int fi = w[l], fo = w[l + 1];
        float bound = float(std::sqrt(6.0 / (fi + fo)));
        for (int i = 0; i < fo * fi; ++i) p[k++] = float(rng.uniform(-double(bound), double(bound)));
        for (int i = 0; i < fo; ++i) p[k++] = 0.f;
    }
}

int level_resolution(const tfg_field_config& c, int l) {
    if (c.levels <= 1) return c.n_min;
    double b = std::exp((std::log(double(c.n_max)) - std::log(double(c.n_min))) /
                        double(c.levels - 1));
    return int(std::floor(c.n_min * std::pow(b, l) + 0.5));
}

cudaEvent_t pool_event(tfg_ctx* c) {
    if (!c->ev_pool.empty()) {
        cudaEvent_t e = c->ev_pool.back();
        c->ev_pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
}
struct PhaseScope {
    tfg_ctx* c;
    int ph;
    cudaEvent_t a = nullptr;
    uint64_t l0;
    PhaseScope(tfg_ctx* c_, int ph_) : c(c_), ph(ph_), l0(c_->launches) {
        if (c->prof) {
            a = pool_event(c);
            cudaEventRecord(a, c->st);
        }
    }
    ~PhaseScope() {
        if (c->prof) {
            cudaEvent_t b = pool_event(c);
            cudaEventRecord(b, c->st);
            c->ev_open.push_back({ph, {a, b}});
        }
        c->prof_launch[ph] += c->launches - l0;
    }
};
void prof_collect(tfg_ctx* c) {
    for (auto& e : c->ev_open) {
        cudaEventSynchronize(e.second.second);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e.second.first, e.second.second);
        c->prof_ms[e.first] += ms;
        c->prof_n[e.first] += 1;
        c->ev_pool.push_back(e.second.first);
        c->ev_pool.push_back(e.second.second);
    }
    c->ev_open.clear();
}

void tile_box(const tfg_ctx* c, int ti, double* b) {
    int r = ti / c->cols, cc = ti % c->cols;
    b[0] = c->east[cc];
    b[1] = c->north[r];
    b[2] = c->roi.z_min;
    b[3] = c->east[cc + 1];
    b[4] = c->north[r + 1];
    b[5] = c->roi.z_max;
}

// crop_for_tile (camera.cpp:126-146) on the host; false when empty/invalid.
bool crop_for_tile(const tfg_rpc& cam, const double* box, int margin, Crop* out) {
    double rlo = HUGE_VAL, rhi = -HUGE_VAL, clo = HUGE_VAL, chi = -HUGE_VAL;
    for (int i = 0; i < 8; ++i) {
        double x = (i & 1) ? box[3] : box[0];
        double y = (i & 2) ? box[4] : box[1];
        double z = (i & 4) ? box[5] : box[2];
        double r, q;
        if (!rpc_project(cam, x, y, z, &r, &q)) return false;
        rlo = std::min(rlo, r);
        rhi = std::max(rhi, r);
        clo = std::min(clo, q);
        chi = std::max(chi, q);
    }
    out->r0 = std::max(0, int(std::floor(rlo)) - margin);
    out->r1 = std::min(cam.image_rows, int(std::ceil(rhi)) + 1 + margin);
    out->c0 = std::max(0, int(std::floor(clo)) - margin);
    out->c1 = std::min(cam.image_cols, int(std::ceil(chi)) + 1 + margin);
    return !out->empty();
}

std::vector<int> window_tiles(const tfg_ctx* c, int pr, int pc) {
    if (c->rows == 1 && c->cols == 1) return {0};
    return {pr * c->cols + pc, pr * c->cols + pc + 1, (pr + 1) * c->cols + pc,
            (pr + 1) * c->cols + pc + 1};
}

// Per view: crop rects of the window's tiles and their union.
void window_crops(const tfg_ctx* c, const std::vector<int>& tl, std::vector<Crop>& crops,
                  std::vector<Crop>& uni) {
    crops.assign(size_t(c->n_views) * kTrainSlots, Crop{});
    uni.assign(c->n_views, Crop{});
    for (int v = 0; v < c->n_views; ++v) {
        Crop u{INT32_MAX, INT32_MIN, INT32_MAX, INT32_MIN};
        bool any = false;
        for (size_t k = 0; k < tl.size(); ++k) {
            double b[6];
            tile_box(c, tl[k], b);
            Crop cr;
            if (!crop_for_tile(c->cams[v], b, c->tc.margin_px, &cr)) continue;
            crops[size_t(v) * kTrainSlots + k] = cr;
            u.r0 = std::min(u.r0, cr.r0);
            u.r1 = std::max(u.r1, cr.r1);
            u.c0 = std::min(u.c0, cr.c0);
            u.c1 = std::max(u.c1, cr.c1);
            any = true;
        }
        uni[v] = any ? u : Crop{};
    }
}

void fresh_tile(tfg_ctx* c, int ti) {
    TileHost& t = c->tiles[ti];
    int row = ti / c->cols, col = ti % c->cols;
    float* p = t.rec;
    Rng re(hash_combine(hash_combine(hash_combine(c->tc.seed, kPurposeTileEnc), uint64_t(row)),
                        uint64_t(col)));
    for (uint64_t i = 0; i < c->enc_n; ++i) p[i] = float(re.uniform(-1e-4, 1e-4));
    Rng rd(hash_combine(hash_combine(hash_combine(c->tc.seed, kPurposeTileDnet), uint64_t(row)),
                        uint64_t(col)));
    const int dw[3] = {kFeatDim, kDHidden, kDOut};
    std::fill(p + c->enc_n, p + c->dn_off, 0.f);  // alignment padding (none by default)
    mlp_init_host(dw, 3, rd, p + c->dn_off);
    std::fill(p + c->dn_off + c->dn_n, p + c->stride, 0.f);
    std::memset(p + c->stride, 0, 2 * c->stride * sizeof(float));
    float* ema = p + 3 * c->stride;
    for (int i = 0; i < kOccVox; ++i) ema[i] = 1.0f;
    t.enc_step = t.dnet_step = 0;
    t.created = true;
}

int ensure_record(tfg_ctx* c, int ti) {
    // the record was created by the init pool (or is being created now)
    while (!c->init.ready[ti].load(std::memory_order_acquire)) std::this_thread::yield();
    return 0;
}

void stop_init_pool(tfg_ctx* c) {
    c->init.stop = true;
    for (auto& w : c->init.workers) w.join();
    c->init.workers.clear();
    c->init.stop = false;
}

void start_init_pool(tfg_ctx* c) {
    int n = c->rows * c->cols;
    c->init.ready.reset(new std::atomic<int>[n]);
    for (int i = 0; i < n; ++i) c->init.ready[i] = 0;
    // first-visit order along the snake path
    std::vector<int> order;
    std::vector<char> seen(n, 0);
    auto visit = [&](int ti) {
        if (!seen[ti]) {
            seen[ti] = 1;
            order.push_back(ti);
        }
    };
    if (c->rows == 1 && c->cols == 1) {
        visit(0);
    } else {
        for (int i = 0; i < c->rows - 1; ++i)
            for (int jj = 0; jj < c->cols - 1; ++jj) {
                int j = (i % 2 == 0) ? jj : (c->cols - 2 - jj);
                for (int ti : window_tiles(c, i, j)) visit(ti);
            }
    }
    for (int ti = 0; ti < n; ++ti) visit(ti);
    c->init.order = order;
    c->init.next = 0;
    int nw = std::max(1u, std::min(8u, std::thread::hardware_concurrency()));
    for (int w = 0; w < nw; ++w)
        c->init.workers.emplace_back([c] {
            for (;;) {
                size_t k = c->init.next.fetch_add(1);
                if (k >= c->init.order.size() || c->init.stop) return;
                int ti = c->init.order[k];
                fresh_tile(c, ti);
                c->init.ready[ti].store(1, std::memory_order_release);
            }
        });
}

// D2H (evict) / H2D (load) of one slot's state on the side stream.
int slot_copy(tfg_ctx* c, int slot, int ti, bool to_host) {
    TileHost& t = c->tiles[ti];
    uint64_t off = uint64_t(slot) * c->stride;
    size_t bytes = c->stride * sizeof(float);
    cudaMemcpyKind k = to_host ? cudaMemcpyDeviceToHost : cudaMemcpyHostToDevice;
    float* dev[3] = {c->d_params + off, c->d_m + off, c->d_v + off};
    (to_host ? c->d2h_bytes : c->h2d_bytes) += 3 * bytes + kOccVox * sizeof(float);
    for (int a = 0; a < 3; ++a) {
        float* h = t.rec + a * c->stride;
        CK(cudaMemcpyAsync(to_host ? static_cast<void*>(h) : static_cast<void*>(dev[a]),
                           to_host ? static_cast<const void*>(dev[a]) : static_cast<const void*>(h),
                           bytes, k, c->side));
    }
    float* de = c->d_ema + uint64_t(slot) * kOccVox;
    float* he = t.rec + 3 * c->stride;
    CK(cudaMemcpyAsync(to_host ? static_cast<void*>(he) : static_cast<void*>(de),
                       to_host ? static_cast<const void*>(de) : static_cast<const void*>(he),
                       kOccVox * sizeof(float), k, c->side));
    return 0;
}

// D2D between a device slot (params / m / v / EMA spans) and a contiguous
// staged record (the host record layout), on stream st.
int slot_record_d2d(tfg_ctx* c, int slot, float* rec, bool to_record, cudaStream_t st) {
    uint64_t off = uint64_t(slot) * c->stride;
    size_t bytes = c->stride * sizeof(float);
    float* dev[4] = {c->d_params + off, c->d_m + off, c->d_v + off, c->d_ema + uint64_t(slot) * kOccVox};
    size_t nb[4] = {bytes, bytes, bytes, kOccVox * sizeof(float)};
    for (int a = 0; a < 4; ++a) {
        float* r = rec + a * c->stride;
        CK(cudaMemcpyAsync(to_record ? static_cast<void*>(r) : static_cast<void*>(dev[a]),
                           to_record ? static_cast<const void*>(dev[a]) : static_cast<const void*>(r), nb[a],
                           cudaMemcpyDeviceToDevice, st));
    }
    return 0;
}

void fill_slots(tfg_ctx* c) {
    c->slots.n = c->nslots;
    for (int k = 0; k < c->nslots; ++k) {
        double b[6];
        tile_box(c, c->slot_tile[k], b);
        for (int q = 0; q < 6; ++q) c->slots.box[k][q] = b[q];
        for (int q = 0; q < 3; ++q) {
            c->slots.frame[k][q] = b[q];
            c->slots.frame[k][3 + q] = 1.0 / (b[3 + q] - b[q]);  // cwiseInverse (tiler.cpp:49)
        }
    }
}

FieldPtrs train_ptrs(tfg_ctx* c) {
    FieldPtrs f{};
    for (int k = 0; k < c->nslots; ++k) {
        f.enc[k] = c->d_params + uint64_t(k) * c->stride;
        f.enc16[k] = static_cast<uint16_t*>(c->d_enc16) + uint64_t(k) * c->enc16_stride;
        f.dnet[k] = f.enc[k] + c->dn_off;
        f.occ_bits[k] = c->d_bits + uint64_t(k) * kOccWords;
    }
    f.color = c->d_params + c->color_off;
    return f;
}

int run_occupancy(tfg_ctx* c, bool update, uint64_t* keys) {
    PhaseScope ps(c, kPhOccupancy);
    OccArgs o{};
    o.hl = c->hl;
    o.density_lim = c->density_lim;
    o.n = c->nslots;
    for (int k = 0; k < c->nslots; ++k) {
        o.enc[k] = c->d_params + uint64_t(k) * c->stride;
        o.dnet[k] = o.enc[k] + c->dn_off;
        o.ema[k] = c->d_ema + uint64_t(k) * kOccVox;
        o.bits[k] = c->d_bits + uint64_t(k) * kOccWords;
        o.base_key[k] = keys ? keys[k] : 0;
    }
    o.decay = c->fc.occupancy_decay;
    o.threshold = c->fc.occupancy_threshold;
    o.density_max = c->fc.density_max;
    o.update = update ? 1 : 0;
    o.sticky = c->d_sticky;
    launch_occupancy(o, c->st, &c->launches);
    CK(cudaGetLastError());
    return 0;
}

// Stages window position (pr, pc) into w on `st`: the union crop of each
// view (2D copies from the pinned images) and the accepted-ray list
// (SPEC.md:437-445).  Independent of the slot assignment.
int stage_window(tfg_ctx* c, WinBuf& w, int pr, int pc, cudaStream_t st) {
    std::vector<int> want = window_tiles(c, pr, pc);
    std::vector<Crop> crops, uni;
    window_crops(c, want, crops, uni);
    w.h_crop_rect.assign(4 * c->n_views, 0);
    w.h_crop_off.assign(c->n_views, 0);
    uint64_t off = 0;
    for (int v = 0; v < c->n_views; ++v) {
        const Crop& u = uni[v];
        w.h_crop_off[v] = off;
        if (u.empty()) continue;
        int cw = u.c1 - u.c0, ch = u.r1 - u.r0;
        w.h_crop_rect[4 * v] = u.r0;
        w.h_crop_rect[4 * v + 1] = u.c0;
        w.h_crop_rect[4 * v + 2] = cw;
        w.h_crop_rect[4 * v + 3] = ch;
        const uint8_t* src = c->h_images[v] + 3 * (size_t(u.r0) * c->cams[v].image_cols + u.c0);
        c->h2d_bytes += uint64_t(cw) * 3 * ch;
        CK(cudaMemcpy2DAsync(w.d_crops + off, size_t(cw) * 3, src, size_t(c->cams[v].image_cols) * 3,
                             size_t(cw) * 3, ch, cudaMemcpyHostToDevice, st));
        off += uint64_t(cw) * ch * 3;
    }
    CK(cudaMemcpyAsync(w.d_crop_rect, w.h_crop_rect.data(), 4 * c->n_views * 4, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(w.d_crop_off, w.h_crop_off.data(), c->n_views * 8, cudaMemcpyHostToDevice, st));
    // accepted-ray list
    std::vector<uint64_t> vs(c->n_views);
    std::vector<int> urect(4 * c->n_views), crect(4 * c->n_views * kTrainSlots, 0);
    uint64_t n = 0;
    for (int v = 0; v < c->n_views; ++v) {
        vs[v] = n;
        const Crop& u = uni[v];
        urect[4 * v] = u.r0;
        urect[4 * v + 1] = u.r1;
        urect[4 * v + 2] = u.c0;
        urect[4 * v + 3] = u.c1;
        if (!u.empty()) n += uint64_t(u.r1 - u.r0) * uint64_t(u.c1 - u.c0);
        else urect[4 * v + 1] = urect[4 * v], urect[4 * v + 3] = urect[4 * v + 2] + 1;
        for (int k = 0; k < kTrainSlots; ++k) {
            const Crop& cr = crops[size_t(v) * kTrainSlots + k];
            int* d = &crect[4 * (v * kTrainSlots + k)];
            d[0] = cr.r0;
            d[1] = cr.r1;
            d[2] = cr.c0;
            d[3] = cr.c1;
        }
    }
    if (n > c->cand_cap) return fail(TFG_ERR_INVALID, "accept: candidate capacity exceeded");
    // synchronous pageable copies: the host vectors may go out of scope
    CK(cudaMemcpyAsync(c->d_view_start, vs.data(), vs.size() * 8, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(c->d_union, urect.data(), urect.size() * 4, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(c->d_crop4, crect.data(), crect.size() * 4, cudaMemcpyHostToDevice, st));
    AcceptArgs a{};
    a.cams = c->d_cams;
    a.loc = c->d_loc;
    a.n_views = c->n_views;
    a.view_start = c->d_view_start;
    a.union_rect = c->d_union;
    a.crop_rect = c->d_crop4;
    a.n_candidates = n;
    a.east = c->d_east;
    a.north = c->d_north;
    a.grid_rows = c->rows;
    a.grid_cols = c->cols;
    for (int k = 0; k < kTrainSlots; ++k) a.loaded_tile[k] = k < int(want.size()) ? want[k] : -1;
    a.n_loaded = int(want.size());
    a.z_min = c->roi.z_min;
    a.z_max = c->roi.z_max;
    // the memo applies when the loaded tiles form a rectangle (every window does)
    {
        int r0 = 1 << 30, r1 = -1, c0 = 1 << 30, c1 = -1;
        for (int ti : want) {
            r0 = std::min(r0, ti / c->cols);
            r1 = std::max(r1, ti / c->cols);
            c0 = std::min(c0, ti % c->cols);
            c1 = std::max(c1, ti % c->cols);
        }
        bool rect = !want.empty() && int(want.size()) == (r1 - r0 + 1) * (c1 - c0 + 1);
        a.win_r0 = r0;
        a.win_r1 = r1;
        a.win_c0 = c0;
        a.win_c1 = c1;
        // the other window buffer holds the previous position (staged earlier
        // on the same side stream): its solved pixels are copied, not re-solved
        const WinBuf& o = (&w == &c->win[0]) ? c->win[1] : c->win[0];
        if (rect && c->memo_reuse && o.pos_r >= 0) {
            a.o_info = o.d_minfo;
            a.o_rays = o.d_mrays;
            a.o_rect = o.d_crop_rect;
            a.o_off = o.d_crop_off;
        }
    }
    a.m_info = w.d_minfo;
    a.m_rays = w.d_mrays;
    a.todo_n = c->d_todo_n;
    a.sms = c->sms;
    if (launch_accept(a, c->d_flags, c->d_pos, c->d_acc_sums, w.d_n, w.d_accept, st, &c->launches))
        return fail(TFG_ERR_INVALID, "accept: scan capacity exceeded");
    CK(cudaGetLastError());
    CK(cudaEventRecord(w.ready, st));
    w.pos_r = pr;
    w.pos_c = pc;
    return 0;
}

uint64_t read_accept_count(tfg_ctx* c) {
    uint32_t n = 0;
    if (cudaMemcpyAsync(&c->h_status->pad, c->win[c->front].d_n, 4, cudaMemcpyDeviceToHost, c->st) !=
            cudaSuccess ||
        cudaStreamSynchronize(c->st) != cudaSuccess)
        return 0;
    n = c->h_status->pad;
    return n;
}

int check_status(tfg_ctx* c) {
    Status& s = *c->h_status;
    if (s.bits & kStatusSampleOverflow)
        return fail(TFG_ERR_INVALID, "sample: batch exceeds the sample capacity of the context");
    if (s.bits & kStatusSegOverflow) return fail(TFG_ERR_INVALID, "sample: more than 8 segments");
    if (s.bits & kStatusBadBatch)
        return fail(TFG_ERR_INVALID, "batch_import: a ray's samples must form at most one run per loaded slot "
                                     "(slot < number of slots; a ray crosses each tile box once)");
    if (s.bits & kStatusRayFail)
        return fail(TFG_ERR_INVALID,
                    "sample: ray generation failed (ray_from_pixel threw for a drawn pixel, or the "
                    "window's accepted-ray list is empty)");
    if (!c->nonfinite_pending.empty()) {
        std::string m = c->nonfinite_pending;
        c->nonfinite_pending.clear();
        return fail(TFG_ERR_NONFINITE, m);
    }
    return 0;
}

// Consumes the sticky non-finite record once (host copy already taken): the
// step-count increments of the failed optimizer step and of every later one
// (skipped on the device as well) are rolled back, the group is named, and
// the record is cleared on the device.
void consume_sticky(tfg_ctx* c, const uint32_t* k, uint32_t upto_seq) {
    if (k[0] && k[2] != c->sticky_done_seq) {
        const uint32_t g = k[1], seq = k[2];
        char nm[96];
        std::snprintf(nm, sizeof nm, "color");
        for (auto it = c->unverified.rbegin(); it != c->unverified.rend(); ++it) {
            if (int32_t(it->seq - seq) < 0) break;
            for (int s = 0; s < it->nslots; ++s) {
                TileHost& th = c->tiles[it->tile[s]];
                --th.enc_step;
                --th.dnet_step;
            }
            --c->color_step;
            if (it->seq == seq && int(g) < 2 * it->nslots) {
                int ti = it->tile[g / 2];
                std::snprintf(nm, sizeof nm, "tile(%d,%d).%s", ti / c->cols, ti % c->cols, (g % 2) ? "dnet" : "enc");
            }
        }
        c->nonfinite_pending = std::string("adam_step: non-finite gradient in group ") + nm;
        c->sticky_done_seq = seq;
        cudaMemsetAsync(c->d_sticky, 0, 16, c->st);
        // every step from the failing one on was skipped (and is rolled back),
        // the earlier ones were applied
        c->unverified.clear();
        return;
    }
    // no new failure up to the snapshot: the steps it covers are final
    auto& u = c->unverified;
    u.erase(std::remove_if(u.begin(), u.end(), [&](const tfg_ctx::StepRec& r) { return int32_t(r.seq - upto_seq) <= 0; }),
            u.end());
}
void consume_sticky(tfg_ctx* c) { consume_sticky(c, c->h_sticky, c->step_seq); }

// Reads the sticky record (synchronises) and settles the unverified steps.
int settle_steps(tfg_ctx* c) {
    CK(cudaMemcpyAsync(c->h_sticky, c->d_sticky, 16, cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
    consume_sticky(c);
    return 0;
}

int sync_status(tfg_ctx* c) {
    c->d2h_bytes += sizeof(Status) + 16;
    CK(cudaMemcpyAsync(c->h_status, c->d_status, sizeof(Status), cudaMemcpyDeviceToHost, c->st));
    CK(cudaMemcpyAsync(c->h_sticky, c->d_sticky, 16, cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
    consume_sticky(c);
    return check_status(c);
}

RaygenArgs base_raygen(tfg_ctx* c) {
    RaygenArgs a{};
    a.cams = c->d_cams;
    a.loc = c->d_loc;
    a.seed = c->tc.seed;
    a.z_min = c->roi.z_min;
    a.z_max = c->roi.z_max;
    a.spm = c->tc.samples_per_meter;
    a.cap = c->tc.max_samples_per_ray;
    a.delta_cap = c->tc.delta_cap;
    a.slots = c->slots;
    for (int k = 0; k < c->nslots; ++k) a.occ_bits[k] = c->d_bits + uint64_t(k) * kOccWords;
    const WinBuf& w = c->win[c->front];
    a.crop_bytes = w.d_crops;
    a.crop_rect = w.d_crop_rect;
    a.crop_offset = w.d_crop_off;
    return a;
}

int run_sampler(tfg_ctx* c, RaygenArgs& a) {
    if (a.n_rays <= 0 || a.n_rays > c->max_rays)
        return fail(TFG_ERR_INVALID, "sample: n_rays outside (0, max_rays]");
    PhaseScope ps(c, kPhSampler);
    CK(cudaMemsetAsync(c->d_status, 0, sizeof(Status), c->st));
    if (launch_sampler(a, c->d_rays, c->d_hdr, c->d_venc, c->d_counts, c->d_P, c->d_block_sums, c->d_tiles,
                       c->max_tiles, c->s, c->sample_cap, c->d_status, c->st, &c->launches))
        return fail(TFG_ERR_INVALID, "sample: scan capacity exceeded");
    CK(cudaGetLastError());
    c->cur_rays = a.n_rays;
    c->have_batch = true;
    c->fwd_done = false;
    return 0;
}

FieldArgs field_args(tfg_ctx* c, const FieldPtrs& f) {
    FieldArgs a{};
    a.f = f;
    a.hl = c->hl;
    a.density_max = c->fc.density_max;
    a.density_lim = c->density_lim;
    a.tiles = c->d_tiles;
    a.status = c->d_status;
    a.venc = c->d_venc;
    a.s = c->s;
    return a;
}

int run_forward(tfg_ctx* c, const FieldPtrs& f) {
    PhaseScope ps(c, kPhFieldFwd);
    if (!c->render_mode && c->enc16_dirty && c->nslots > 0) {  // slot tables written outside Adam
        launch_enc_half(c->d_params, c->stride, c->nslots, c->enc_n, c->enc16_stride, c->d_enc16, c->st,
                        &c->launches);
        c->enc16_dirty = false;
    }
    c->fwd_done = true;
    c->io_fwd = true;
    launch_field_forward_tc(field_args(c, f), c->d_feat, c->d_tile_rays, c->sms, c->st,
                            &c->launches);
    CK(cudaGetLastError());
    return 0;
}

int run_composite(tfg_ctx* c, bool backward, float4* export_io = nullptr) {
    PhaseScope ps(c, kPhComposite);
    if (backward) c->io_fwd = false;  // io now holds the pre-activation gradients
    CompositeArgs a{};
    a.hdr = c->d_hdr;
    a.n_rays = c->cur_rays;
    a.sms = c->sms;
    a.s = c->s;
    a.status_in = c->d_status;
    a.status = c->d_status;
    a.bg = make_float3(c->tc.background[0], c->tc.background[1], c->tc.background[2]);
    a.inv3b = 1.0f / (3.0f * float(c->tc.batch_rays));
    a.backward = backward ? 1 : 0;
    a.ray_rgb = c->d_ray_out;
    a.ray_depth = c->d_ray_out + 3 * uint64_t(c->max_rays);
    a.ray_opacity = c->d_ray_out + 4 * uint64_t(c->max_rays);
    a.density_max = c->fc.density_max;
    a.export_io = export_io;
    a.loss_parts = c->d_loss_parts;
    launch_composite(a, c->st, &c->launches);
    CK(cudaGetLastError());
    return 0;
}

int run_backward(tfg_ctx* c) {
    // the backward recomputes the forward from the feature tiles of this
    // batch's forward and reads K3's gradients from io
    if (!c->fwd_done) return fail(TFG_ERR_STATE, "field_backward: run field_forward on this batch first");
    PhaseScope ps(c, kPhFieldBwd);
    CK(cudaMemsetAsync(c->d_grads, 0, c->n_params * sizeof(float), c->st));
    FieldGradArgs g{};
    for (int k = 0; k < c->nslots; ++k) {
        g.g_enc[k] = c->d_grads + uint64_t(k) * c->stride;
        g.g_dnet[k] = g.g_enc[k] + c->dn_off;
    }
    g.g_color = c->d_grads + c->color_off;
    launch_field_backward_tc(field_args(c, train_ptrs(c)), g, c->d_feat, c->d_tile_rays,
                             c->sms, c->st, &c->launches);
    CK(cudaGetLastError());
    return 0;
}

// Per-sample host reorder: bucket order -> ray order (RaySegmentBatch layout).
struct HostBatch {
    std::vector<RayRec> rays;
    std::vector<uint32_t> P;
    uint64_t n_samples = 0;
    // occupied [lo, hi) of each slot bucket in the device sample arrays and
    // the extent they span
    std::vector<std::pair<uint64_t, uint64_t>> ranges;
    uint64_t extent = 0;
};
int fetch_batch_meta(tfg_ctx* c, HostBatch& hb) {
    int n = c->cur_rays;
    hb.rays.resize(n);
    uint64_t np = uint64_t(c->slots.n) * n + 1;
    hb.P.resize(np);
    CK(cudaMemcpyAsync(hb.rays.data(), c->d_rays, n * sizeof(RayRec), cudaMemcpyDeviceToHost, c->st));
    CK(cudaMemcpyAsync(hb.P.data(), c->d_P, np * 4, cudaMemcpyDeviceToHost, c->st));
    int st = sync_status(c);
    if (st) return st;
    hb.n_samples = c->h_status->n_samples;
    const int ns = c->slots.n;
    hb.ranges.assign(ns, {UINT64_MAX, 0});
    for (int i = 0; i < n; ++i) {
        const RayRec& R = hb.rays[i];
        if (R.status != 0) continue;
        for (int k = 0; k < R.nseg; ++k) {
            const int sl = R.slot[k];
            const uint64_t b = hb.P[uint64_t(sl) * n + i];
            auto& r = hb.ranges[sl];
            r.first = std::min(r.first, b);
            r.second = std::max(r.second, b + R.cnt[k]);
        }
    }
    hb.extent = 0;
    for (auto& r : hb.ranges) {
        if (r.first > r.second) r = {0, 0};
        hb.extent = std::max(hb.extent, r.second);
    }
    return 0;
}
// Per-sample device array <-> host array indexed like the device (only the
// occupied bucket ranges are copied).
template <typename T>
int pull_samples(const HostBatch& hb, const T* dev, std::unique_ptr<T[]>& host) {
    host.reset(new T[std::max<uint64_t>(1, hb.extent)]);
    for (auto& r : hb.ranges)
        if (r.second > r.first)
            CK(cudaMemcpy(host.get() + r.first, dev + r.first, (r.second - r.first) * sizeof(T), cudaMemcpyDeviceToHost));
    return 0;
}
template <typename T>
int push_samples(const HostBatch& hb, const T* host, T* dev) {
    for (auto& r : hb.ranges)
        if (r.second > r.first)
            CK(cudaMemcpy(dev + r.first, host + r.first, (r.second - r.first) * sizeof(T), cudaMemcpyHostToDevice));
    return 0;
}
// Visits samples in ray order: fn(ray, sample index in ray order, bucket pos, slot).
template <typename F>
void for_samples(const tfg_ctx* c, const HostBatch& hb, F fn) {
    uint64_t q = 0;
    int n = c->cur_rays;
    for (int i = 0; i < n; ++i) {
        const RayRec& R = hb.rays[i];
        if (R.status != 0) continue;
        for (int k = 0; k < R.nseg; ++k) {
            uint64_t base = hb.P[uint64_t(R.slot[k]) * n + i];
            for (int j = 0; j < R.cnt[k]; ++j) fn(i, q++, base + j, int(R.slot[k]));
        }
    }
}

} // namespace host
} // namespace tfg

extern "C" {

TFG_API const char* tfg_last_error(void) { return g_err.c_str(); }

TFG_API int tfg_default_field_config(tfg_field_config* o) {
    *o = tfg_field_config{8, 1 << 15, 2, 16, 256, 64, 15, 64, 2, 4, 1e4f, 32, 0.95f, 0.02f, 16};
    return 0;
}

TFG_API int tfg_default_train_config(tfg_train_config* o) {
    std::memset(o, 0, sizeof(*o));
    o->seed = 2;
    o->samples_per_meter = 63.0 / 40.0;
    o->max_samples_per_ray = 1024;
    o->delta_cap = 10.0;
    o->background[0] = o->background[1] = o->background[2] = 0.5f;
    o->margin_px = 4;
    o->lr_field = 1e-2;
    o->lr_color = 1e-3;
    o->lr_decay_rate = 1.0;
    o->lr_decay_steps = 1000;
    o->beta1 = 0.9f;
    o->beta2 = 0.99f;
    o->eps = 1e-15f;
    o->batch_rays = 65536;
    return 0;
}

TFG_API int tfg_param_counts(const tfg_field_config* c, uint64_t* enc, uint64_t* dnet,
                             uint64_t* color) {
    uint64_t tot = 0;
    for (int l = 0; l < c->levels; ++l) {
        uint64_t r = uint64_t(level_resolution(*c, l)) + 1;
        tot += std::min<uint64_t>(r * r * r, uint64_t(c->table_size));
    }
    if (enc) *enc = tot * c->features;
    auto mlp = [](std::vector<int> w) {
        uint64_t n = 0;
        for (size_t l = 0; l + 1 < w.size(); ++l) n += uint64_t(w[l + 1]) * w[l] + w[l + 1];
        return n;
    };
    if (dnet) *dnet = mlp({c->levels * c->features, c->density_hidden, 1 + c->embedding});
    std::vector<int> cw{c->embedding + 6 * c->view_freqs};
    for (int i = 0; i < c->color_layers; ++i) cw.push_back(c->color_hidden);
    cw.push_back(3);
    if (color) *color = mlp(cw);
    return 0;
}

TFG_API int tfg_create(const tfg_field_config* fcfg, const tfg_train_config* tcfg, int device,
                       int max_rays, tfg_ctx** out) {
    if (!fcfg || !tcfg || !out || max_rays <= 0) return fail(TFG_ERR_INVALID, "create: bad arguments");
    tfg_field_config d;
    tfg_default_field_config(&d);
    // The hash-grid geometry (n_min, n_max, table_size) is free; the feature
    // and MLP widths are the UMMA tile shapes and TMEM column maps of the
    // tensor-core kernels, and the occupancy grid is 32^3 bit words.
    if (fcfg->levels != d.levels || fcfg->features != d.features || fcfg->density_hidden != d.density_hidden ||
        fcfg->embedding != d.embedding || fcfg->color_hidden != d.color_hidden ||
        fcfg->color_layers != d.color_layers || fcfg->view_freqs != d.view_freqs ||
        fcfg->occupancy_resolution != d.occupancy_resolution)
        return fail(TFG_ERR_INVALID, "create: the sm_100a kernels are specialised for the default "
                                     "FieldConfig widths (levels 8, features 2, MLPs 16-64-16 / "
                                     "39-64-64-3, view_freqs 4, occupancy 32^3; nn.hpp:14-37); "
                                     "n_min, n_max and table_size are free");
    if (fcfg->table_size < 16 || fcfg->table_size > (1 << 22) ||
        (fcfg->table_size & (fcfg->table_size - 1)) != 0)
        return fail(TFG_ERR_INVALID, "create: table_size must be a power of two in [2^4, 2^22]");
    if (fcfg->n_min < 1 || fcfg->n_max < fcfg->n_min || fcfg->n_max > (1 << 16))
        return fail(TFG_ERR_INVALID, "create: need 1 <= n_min <= n_max <= 65536");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0 || device >= ndev)
        return fail(TFG_ERR_NO_DEVICE, "create: no CUDA device (there is no CPU fallback)");
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10)
        return fail(TFG_ERR_NO_DEVICE, std::string("create: needs an sm_100 device, found ") + prop.name);
    CK(cudaSetDevice(device));
    auto* c = new tfg_ctx();
    c->device = device;
    c->sms = prop.multiProcessorCount;
    c->fc = *fcfg;
    c->tc = *tcfg;
    c->max_rays = max_rays;
    uint64_t enc, dn, col;
    tfg_param_counts(fcfg, &enc, &dn, &col);
    c->enc_n = enc;
    c->dn_n = dn;
    c->dn_off = (enc + 3) & ~uint64_t(3);
    c->stride = (c->dn_off + dn + 3) & ~uint64_t(3);
    c->enc16_stride = c->dn_off;
    c->color_off = kTrainSlots * c->stride;
    c->n_params = c->color_off + col;
    uint32_t off = 0;
    const uint64_t T = uint64_t(fcfg->table_size);
    for (int l = 0; l < kLevels; ++l) {
        int r = level_resolution(*fcfg, l);
        uint64_t dense = uint64_t(r + 1) * (r + 1) * (r + 1);
        c->hl.res[l] = r;
        c->hl.off[l] = off;
        c->hl.dense[l] = dense <= T ? 1 : 0;
        off += uint32_t(std::min<uint64_t>(dense, T));
    }
    c->hl.mask = uint32_t(T - 1);
    {
        // the default layout is folded into the hash kernels as constants;
        // any other runs their runtime-layout instantiations
        // (TFG_GENERIC_HASH=1 forces those for the default one: a test hook)
        const int res[kLevels] = {16, 24, 35, 53, 78, 116, 172, 256};
        const uint32_t off0[kLevels] = {0, 4913, 20538, 53306, 86074, 118842, 151610, 184378};
        bool same = T == uint64_t(kTable);
        for (int l = 0; l < kLevels; ++l) same = same && c->hl.res[l] == res[l] && c->hl.off[l] == off0[l];
        const char* force = std::getenv("TFG_GENERIC_HASH");
        c->hl.generic = (!same || (force && force[0] == '1')) ? 1 : 0;
    }
    c->density_lim = std::log(fcfg->density_max);
    c->sample_cap = uint64_t(max_rays) * 128;
    c->max_tiles = int(c->sample_cap / 128 + kMaxSlots + 1);
    // everything below may fail part-way: tfg_destroy releases what was made
    auto init = [&]() -> int {
        int rc = 0;
        CK(cudaStreamCreateWithFlags(&c->st, cudaStreamNonBlocking));
        CK(cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&c->ev_main, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&c->ev_side, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&c->ev_swap, cudaEventDisableTiming));
        CK(cudaEventRecord(c->ev_swap, c->st));
        for (cudaEvent_t* e : {&c->ev_stage_in, &c->ev_stage_read, &c->ev_out_done}) {
            CK(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
            CK(cudaEventRecord(*e, c->st));
        }
        rc |= dalloc(c, &c->d_params, c->n_params);
        rc |= dalloc(c, &c->d_stage_in, uint64_t(kTrainSlots) * (3 * c->stride + kOccVox));
        rc |= dalloc(c, &c->d_stage_out, uint64_t(kTrainSlots) * (3 * c->stride + kOccVox));
        rc |= dalloc(c, &c->d_grads, c->n_params);
        rc |= dalloc(c, &c->d_m, c->n_params);
        rc |= dalloc(c, &c->d_v, c->n_params);
        rc |= dalloc(c, &c->d_ema, uint64_t(kTrainSlots) * kOccVox);
        rc |= dalloc(c, &c->d_bits, uint64_t(kMaxSlots) * kOccWords);
        rc |= dalloc(c, reinterpret_cast<uint16_t**>(&c->d_enc16), uint64_t(kTrainSlots + kMaxSlots) * c->enc16_stride);
        rc |= dalloc(c, &c->d_group_flags, 16);
        rc |= dalloc(c, &c->d_sticky, 4);
        rc |= dalloc(c, &c->d_status, 1);
        rc |= dalloc(c, &c->d_rays, max_rays);
        rc |= dalloc(c, &c->d_hdr, max_rays);
        rc |= dalloc(c, &c->d_venc, uint64_t(max_rays) * 6);
        rc |= dalloc(c, &c->d_counts, uint64_t(max_rays) * kMaxSlots);
        rc |= dalloc(c, &c->d_P, uint64_t(max_rays) * kMaxSlots + 1);
        rc |= dalloc(c, &c->d_tiles, c->max_tiles);
        rc |= dalloc(c, &c->s.local, c->sample_cap);
        rc |= dalloc(c, &c->s.td, c->sample_cap);
        rc |= dalloc(c, &c->s.endpoint, c->sample_cap);
        rc |= dalloc(c, &c->s.io, c->sample_cap);
        rc |= dalloc(c, &c->d_ray_out, uint64_t(max_rays) * 5);
        rc |= dalloc(c, &c->d_pixels, uint64_t(max_rays) * 3);
        rc |= dalloc(c, &c->d_feat, uint64_t(c->max_tiles) * 4096);
        rc |= dalloc(c, &c->d_loss_parts, uint64_t(max_rays) / 8 + 1);
        rc |= dalloc(c, &c->d_tile_rays, uint64_t(c->max_tiles) * 128);
        rc |= dalloc(c, &c->d_block_sums, 4096 + 64);
        rc |= dalloc(c, &c->d_acc_sums, 4096 + 64);
        rc |= dalloc(c, &c->d_todo_n, 1);
        rc |= dalloc(c, &c->d_rcam, 1);
        rc |= dalloc(c, &c->d_rloc, 2);
        if (rc) return TFG_ERR_CUDA;
        CK(cudaHostAlloc(reinterpret_cast<void**>(&c->h_status), sizeof(Status), cudaHostAllocDefault));
        CK(cudaHostAlloc(reinterpret_cast<void**>(&c->h_sticky), 16, cudaHostAllocDefault));
        CK(cudaMemsetAsync(c->d_sticky, 0, 16, c->st));
        CK(cudaMemsetAsync(c->d_params, 0, c->n_params * 4, c->st));
        CK(cudaMemsetAsync(c->d_m, 0, c->n_params * 4, c->st));
        CK(cudaMemsetAsync(c->d_v, 0, c->n_params * 4, c->st));
        CK(cudaMemsetAsync(c->d_grads, 0, c->n_params * 4, c->st));
        CK(cudaMemsetAsync(c->d_status, 0, sizeof(Status), c->st));
        // GlobalColorNet::create (field.hpp:118)
        std::vector<float> color(col);
        Rng rcn(hash_combine(c->tc.seed, kPurposeColor));
        const int cw[4] = {kCIn, kCHidden, kCHidden, 3};
        mlp_init_host(cw, 4, rcn, color.data());
        CK(cudaMemcpyAsync(c->d_params + c->color_off, color.data(), col * 4, cudaMemcpyHostToDevice, c->st));
        CK(cudaStreamSynchronize(c->st));
        return 0;
    };
    int rc = init();
    if (rc) {
        std::string msg = g_err;
        tfg_destroy(c);
        g_err = msg;
        return rc;
    }
    *out = c;
    return 0;
}

TFG_API int tfg_destroy(tfg_ctx* c) {
    if (!c) return 0;
    cudaSetDevice(c->device);
    cudaDeviceSynchronize();
    comm_release(c);
    void* dev[] = {c->d_params, c->d_grads, c->d_m, c->d_v, c->d_ema, c->d_bits, c->d_group_flags, c->d_sticky,
                   c->d_enc16,
                   c->d_status, c->d_cams, c->d_east, c->d_north, c->d_flags, c->d_pos,
                   c->d_block_sums, c->d_acc_sums, c->d_todo_n, c->d_view_start, c->d_union, c->d_crop4,
                   c->d_rays, c->d_hdr, c->d_venc,
                   c->d_counts, c->d_P, c->d_tiles, c->s.local, c->s.td, c->s.endpoint, c->s.io,
                   c->d_ray_out, c->d_pixels, c->d_rparams, c->d_rbits, c->d_rcolor, c->d_rcam, c->d_rloc, c->d_loc,
                   c->d_feat, c->d_tile_rays, c->d_export,
                   c->d_stage_in, c->d_stage_out, c->d_loss_parts, c->d_imp};
    for (void* p : dev)
        if (p) cudaFree(p);
    stop_init_pool(c);
    if (c->h_records) cudaFreeHost(c->h_records);
    for (auto* im : c->h_images)
        if (im) cudaFreeHost(im);
    if (c->h_status) cudaFreeHost(c->h_status);
    if (c->h_sticky) cudaFreeHost(c->h_sticky);
    if (c->h_ring) cudaFreeHost(c->h_ring);
    if (c->h_ring_sticky) cudaFreeHost(c->h_ring_sticky);
    for (cudaEvent_t e : c->ev_ring)
        if (e) cudaEventDestroy(e);
    for (void* p : {static_cast<void*>(c->h_rpix), static_cast<void*>(c->h_rout), static_cast<void*>(c->h_rstat)})
        if (p) cudaFreeHost(p);
    for (cudaEvent_t e : c->ev_rdone)
        if (e) cudaEventDestroy(e);
    for (WinBuf& w : c->win) {
        void* wo[] = {w.d_crops, w.d_crop_rect, w.d_crop_off, w.d_accept, w.d_n, w.d_minfo, w.d_mrays};
        for (void* p : wo)
            if (p) cudaFree(p);
        if (w.ready) cudaEventDestroy(w.ready);
    }
    if (c->ev_swap) cudaEventDestroy(c->ev_swap);
    for (cudaEvent_t e : {c->ev_stage_in, c->ev_stage_read, c->ev_out_done})
        if (e) cudaEventDestroy(e);
    if (c->ev_main) cudaEventDestroy(c->ev_main);
    if (c->ev_side) cudaEventDestroy(c->ev_side);
    if (c->side) cudaStreamDestroy(c->side);
    if (c->own_stream && c->st) cudaStreamDestroy(c->st);
    delete c;
    return 0;
}

TFG_API int tfg_set_stream(tfg_ctx* c, void* stream) {
    if (!c) return fail(TFG_ERR_INVALID, "set_stream: null context");
    CK(cudaStreamSynchronize(c->st));
    if (c->own_stream && c->st) cudaStreamDestroy(c->st);
    c->st = static_cast<cudaStream_t>(stream);
    c->own_stream = false;
    return 0;
}

TFG_API int tfg_set_scene(tfg_ctx* c, const tfg_rpc* cams, int n_views,
                          const uint8_t* const* images, const tfg_roi* roi, int grid_rows,
                          int grid_cols) {
    if (!c || !cams || n_views <= 0 || !roi || grid_rows < 1 || grid_cols < 1)
        return fail(TFG_ERR_INVALID, "set_scene: bad arguments");
    if (!(roi->easting_max > roi->easting_min) || !(roi->northing_max > roi->northing_min) ||
        !(roi->z_max > roi->z_min))
        return fail(TFG_ERR_INVALID, "Roi: extents must be positive and z_max > z_min");
    if ((grid_rows == 1) != (grid_cols == 1))
        return fail(TFG_ERR_INVALID, "set_scene: 1xN grids need the experimental 1x2 window");
    CK(cudaSetDevice(c->device));
    // pending copies (e.g. an evicted tile's asynchronous D2H) target buffers
    // that are about to be freed
    CK(cudaStreamSynchronize(c->side));
    CK(cudaStreamSynchronize(c->st));
    c->n_views = n_views;
    c->cams.assign(cams, cams + n_views);
    c->roi = *roi;
    c->rows = grid_rows;
    c->cols = grid_cols;
    // grid_edges (tiler.cpp:18-27): bit-identical shared edges
    auto edges = [](double lo, double hi, int n) {
        std::vector<double> e(n + 1);
        double step = (hi - lo) / n;
        for (int k = 0; k <= n; ++k) e[k] = lo + k * step;
        e[0] = lo;
        e[n] = hi;
        return e;
    };
    c->east = edges(roi->easting_min, roi->easting_max, grid_cols);
    c->north = edges(roi->northing_min, roi->northing_max, grid_rows);
    for (auto* im : c->h_images)
        if (im) cudaFreeHost(im);
    c->h_images.assign(n_views, nullptr);
    for (int v = 0; v < n_views; ++v) {
        size_t nb = size_t(cams[v].image_rows) * cams[v].image_cols * 3;
        CK(cudaHostAlloc(reinterpret_cast<void**>(&c->h_images[v]), nb, cudaHostAllocDefault));
        if (images && images[v]) std::memcpy(c->h_images[v], images[v], nb);
        else std::memset(c->h_images[v], 0, nb);
    }
    stop_init_pool(c);
    if (c->h_records) cudaFreeHost(c->h_records);
    c->h_records = nullptr;
    c->tiles.assign(size_t(grid_rows) * grid_cols, TileHost{});
    {
        uint64_t rec = 3 * c->stride + kOccVox;
        CK(cudaHostAlloc(reinterpret_cast<void**>(&c->h_records),
                         c->tiles.size() * rec * sizeof(float), cudaHostAllocDefault));
        for (size_t ti = 0; ti < c->tiles.size(); ++ti) c->tiles[ti].rec = c->h_records + ti * rec;
    }
    // capacities: max over all window positions (constant HBM across the snake)
    uint64_t cand = 1, cropb = 1;
    std::vector<std::pair<int, int>> pos;
    if (grid_rows == 1) pos.push_back({0, 0});
    else
        for (int i = 0; i + 1 < grid_rows; ++i)
            for (int j = 0; j + 1 < grid_cols; ++j) pos.push_back({i, j});
    std::vector<Crop> crops, uni;
    for (auto& p : pos) {
        window_crops(c, window_tiles(c, p.first, p.second), crops, uni);
        uint64_t n = 0;
        for (auto& u : uni)
            if (!u.empty()) n += uint64_t(u.r1 - u.r0) * uint64_t(u.c1 - u.c0);
        cand = std::max(cand, n);
        cropb = std::max(cropb, 3 * n);
    }
    c->cand_cap = cand;
    c->accept_cap = cand;
    c->crop_cap = cropb;
    int rc = 0;
    dfree(c, c->d_cams);
    dfree(c, c->d_loc);
    dfree(c, c->d_east);
    dfree(c, c->d_north);
    dfree(c, c->d_flags);
    dfree(c, c->d_pos);
    dfree(c, c->d_view_start);
    dfree(c, c->d_union);
    dfree(c, c->d_crop4);
    rc |= dalloc(c, &c->d_cams, n_views);
    rc |= dalloc(c, &c->d_loc, 2 * uint64_t(n_views));
    rc |= dalloc(c, &c->d_east, grid_cols + 1);
    rc |= dalloc(c, &c->d_north, grid_rows + 1);
    // per window buffer: crops, accepted list and the pixel memo of the crop
    // union (52 B per candidate pixel), all sized by the largest window union
    // over the positions: independent of the ROI / grid size
    for (WinBuf& w : c->win) {
        dfree(c, w.d_crops);
        dfree(c, w.d_crop_rect);
        dfree(c, w.d_crop_off);
        dfree(c, w.d_accept);
        dfree(c, w.d_n);
        dfree(c, w.d_minfo);
        dfree(c, w.d_mrays);
        rc |= dalloc(c, &w.d_crops, c->crop_cap);
        rc |= dalloc(c, &w.d_crop_rect, 4 * n_views);
        rc |= dalloc(c, &w.d_crop_off, n_views);
        rc |= dalloc(c, &w.d_accept, c->accept_cap);
        rc |= dalloc(c, &w.d_n, 1);
        rc |= dalloc(c, &w.d_minfo, c->cand_cap);
        rc |= dalloc(c, &w.d_mrays, 6 * c->cand_cap);
        if (!w.ready) CK(cudaEventCreateWithFlags(&w.ready, cudaEventDisableTiming));
        w.pos_r = w.pos_c = -1;
    }
    rc |= dalloc(c, &c->d_flags, c->cand_cap);
    rc |= dalloc(c, &c->d_pos, c->cand_cap + 1);
    rc |= dalloc(c, &c->d_view_start, n_views);
    rc |= dalloc(c, &c->d_union, 4 * n_views);
    rc |= dalloc(c, &c->d_crop4, 4 * n_views * kTrainSlots);
    if (rc) return TFG_ERR_CUDA;
    {
        const char* off_env = std::getenv("TFG_NO_MEMO_REUSE");  // A/B + the reuse-off parity test
        // the memo's hit-tile bbox has 7 bits per coordinate
        c->memo_reuse = grid_rows <= 128 && grid_cols <= 128 && !(off_env && off_env[0] == '1');
    }
    CK(cudaMemcpyAsync(c->d_cams, c->cams.data(), n_views * sizeof(tfg_rpc), cudaMemcpyHostToDevice, c->st));
    launch_loc_start(c->d_cams, n_views, c->roi.z_min, c->roi.z_max, c->d_loc, c->st);
    CK(cudaMemcpyAsync(c->d_east, c->east.data(), (grid_cols + 1) * 8, cudaMemcpyHostToDevice, c->st));
    CK(cudaMemcpyAsync(c->d_north, c->north.data(), (grid_rows + 1) * 8, cudaMemcpyHostToDevice, c->st));
    CK(cudaStreamSynchronize(c->st));
    c->nslots = 0;
    for (int k = 0; k < kTrainSlots; ++k) c->stage_tile[k] = -1;
    c->pos_r = c->pos_c = -1;
    start_init_pool(c);
    return 0;
}

// ---------------------------------------------------------------- window slide
TFG_API int tfg_snake_path(int H, int W, int32_t* out, int* n_out) {
    if (H < 2 || W < 2) return fail(TFG_ERR_INVALID, "snake_path: H and W must be >= 2");
    int m = 0;
    for (int i = 0; i < H - 1; ++i)
        for (int jj = 0; jj < W - 1; ++jj) {
            int j = (i % 2 == 0) ? jj : (W - 2 - jj);
            if (out) {
                out[2 * m] = i;
                out[2 * m + 1] = j;
            }
            ++m;
        }
    if (n_out) *n_out = m;
    return 0;
}

// advance: staying tiles keep their slot; an entering tile
// takes the slot of the leaving tile in the same row (east/west move) or the
// same column (north move).  Leaving tiles are copied to their pinned host
// records and entering ones loaded (fresh TileField::create if never trained)
// on the side stream; then the window crops are staged and the accepted-ray
// list rebuilt.
TFG_API int tfg_set_window(tfg_ctx* c, int pr, int pc) {
    if (!c || c->n_views == 0) return fail(TFG_ERR_STATE, "set_window: call set_scene first");
    CK(cudaSetDevice(c->device));
    bool single = (c->rows == 1 && c->cols == 1);
    if (!single && (pr < 0 || pc < 0 || pr + 1 >= c->rows || pc + 1 >= c->cols))
        return fail(TFG_ERR_INVALID, "set_window: position outside the (H-1)x(W-1) lattice");
    std::vector<int> want = window_tiles(c, single ? 0 : pr, single ? 0 : pc);
    int ns = int(want.size());
    int next[kTrainSlots] = {-1, -1, -1, -1};
    if (c->nslots == ns && ns == kTrainSlots) {
        bool used[kTrainSlots] = {false, false, false, false};
        for (int k = 0; k < ns; ++k)
            for (int s = 0; s < ns; ++s)
                if (c->slot_tile[s] == want[k]) {
                    next[s] = want[k];
                    used[k] = true;
                }
        bool horiz = (pr == c->pos_r);
        for (int k = 0; k < ns; ++k) {
            if (used[k]) continue;
            int wr = want[k] / c->cols, wc = want[k] % c->cols, best = -1;
            for (int s = 0; s < ns; ++s) {
                if (next[s] != -1) continue;
                int lr = c->slot_tile[s] / c->cols, lc = c->slot_tile[s] % c->cols;
                if ((horiz && lr == wr) || (!horiz && lc == wc)) {
                    best = s;
                    break;
                }
            }
            if (best < 0)
                for (int s = 0; s < ns; ++s)
                    if (next[s] == -1) {
                        best = s;
                        break;
                    }
            next[best] = want[k];
        }
    } else {
        for (int k = 0; k < ns; ++k) next[k] = want[k];
    }
    // Entering tiles staged by prefetch_window move in by D2D on the main
    // stream (the evicted state goes out the same way and reaches its host
    // record asynchronously); any other slot change copies through the side
    // stream, which the main stream then waits for.
    const uint64_t rec_n = 3 * c->stride + kOccVox;
    int staged_k[kTrainSlots] = {-1, -1, -1, -1};
    bool any_staged = false, any_plain = false;
    for (int s = 0; s < ns; ++s) {
        bool stays = (s < c->nslots && c->slot_tile[s] == next[s]);
        if (stays) continue;
        for (int k = 0; k < kTrainSlots; ++k)
            if (c->stage_tile[k] == next[s]) staged_k[s] = k;
        if (staged_k[s] >= 0 && s < c->nslots) any_staged = true;
        else staged_k[s] = -1, any_plain = true;
    }
    // main-stream work on the old window must finish before its state moves
    CK(cudaEventRecord(c->ev_main, c->st));
    CK(cudaStreamWaitEvent(c->side, c->ev_main, 0));
    std::vector<std::pair<int, int>> evicted;  // (out record index, tile)
    if (any_staged) {
        CK(cudaStreamWaitEvent(c->st, c->ev_out_done, 0));  // out records free
        CK(cudaStreamWaitEvent(c->st, c->ev_stage_in, 0));  // staged records complete
        for (int s = 0; s < ns; ++s) {
            if (staged_k[s] < 0) continue;
            int old = c->slot_tile[s];
            if (slot_record_d2d(c, s, c->d_stage_out + uint64_t(s) * rec_n, true, c->st)) return TFG_ERR_CUDA;
            evicted.push_back({s, old});
            if (slot_record_d2d(c, s, c->d_stage_in + uint64_t(staged_k[s]) * rec_n, false, c->st))
                return TFG_ERR_CUDA;
            c->h2d_bytes += rec_n * sizeof(float);  // (staged ahead by prefetch_window)
        }
        CK(cudaEventRecord(c->ev_stage_read, c->st));
    }
    for (int k = 0; k < kTrainSlots; ++k) c->stage_tile[k] = -1;
    for (int s = 0; s < c->nslots; ++s) {
        int old = c->slot_tile[s];
        if (old >= 0 && (s >= ns || next[s] != old) && !(s < ns && staged_k[s] >= 0)) {
            if (slot_copy(c, s, old, true)) return TFG_ERR_CUDA;
        }
    }
    for (int s = 0; s < ns; ++s) {
        bool stays = (s < c->nslots && c->slot_tile[s] == next[s]);
        if (stays || staged_k[s] >= 0) continue;
        if (ensure_record(c, next[s])) return TFG_ERR_CUDA;
        if (slot_copy(c, s, next[s], false)) return TFG_ERR_CUDA;
    }
    (void)any_plain;
    for (int s = 0; s < ns; ++s) c->slot_tile[s] = next[s];
    c->enc16_dirty = true;
    c->nslots = ns;
    c->pos_r = pr;
    c->pos_c = pc;
    fill_slots(c);
    // window crops + accepted-ray list: use the prefetched back buffer when it
    // holds this position, else stage it now
    WinBuf& back = c->win[c->front ^ 1];
    if (back.pos_r != pr || back.pos_c != pc) {
        CK(cudaStreamWaitEvent(c->side, c->ev_swap, 0));
        int rc = stage_window(c, back, pr, pc, c->side);
        if (rc) return rc;
    }
    CK(cudaEventRecord(c->ev_side, c->side));
    if (!evicted.empty()) {
        // evicted records: D2H behind the main stream's D2D, off the critical path
        CK(cudaStreamWaitEvent(c->side, c->ev_stage_read, 0));
        for (auto& e : evicted) {
            CK(cudaMemcpyAsync(c->tiles[e.second].rec, c->d_stage_out + uint64_t(e.first) * rec_n,
                               rec_n * sizeof(float), cudaMemcpyDeviceToHost, c->side));
            c->d2h_bytes += rec_n * sizeof(float);
        }
        CK(cudaEventRecord(c->ev_out_done, c->side));
    }
    CK(cudaStreamWaitEvent(c->st, c->ev_side, 0));
    CK(cudaStreamWaitEvent(c->st, back.ready, 0));
    c->front ^= 1;
    // kernels issued from here on use the new front; the old one may be restaged
    CK(cudaEventRecord(c->ev_swap, c->st));
    // host steps of the slots are kept in the tile records (never reset)
    if (run_occupancy(c, false, nullptr)) return TFG_ERR_CUDA;
    c->have_batch = false;
    return 0;
}

// Stages the next window position (crops + accepted-ray list) into the back
// buffer on the side stream while the current position trains; the entering
// tiles' host records are materialised by the init pool.
TFG_API int tfg_prefetch_window(tfg_ctx* c, int pr, int pc) {
    if (!c || c->n_views == 0) return fail(TFG_ERR_STATE, "prefetch_window: call set_scene first");
    CK(cudaSetDevice(c->device));
    bool single = (c->rows == 1 && c->cols == 1);
    if (!single && (pr < 0 || pc < 0 || pr + 1 >= c->rows || pc + 1 >= c->cols))
        return fail(TFG_ERR_INVALID, "prefetch_window: position outside the (H-1)x(W-1) lattice");
    WinBuf& back = c->win[c->front ^ 1];
    if (back.pos_r == pr && back.pos_c == pc) return 0;
    back.pos_r = back.pos_c = -1;
    // entering tiles first: their host records (final while not resident) go
    // to the staging records, so the move itself only does D2D copies
    if (c->nslots == kTrainSlots) {
        std::vector<int> want = window_tiles(c, single ? 0 : pr, single ? 0 : pc);
        const uint64_t rec_n = 3 * c->stride + kOccVox;
        CK(cudaStreamWaitEvent(c->side, c->ev_stage_read, 0));  // previous staged records consumed
        for (int k = 0; k < kTrainSlots; ++k) c->stage_tile[k] = -1;
        int k = 0;
        for (int ti : want) {
            bool resident = false;
            for (int s = 0; s < c->nslots; ++s) resident |= (c->slot_tile[s] == ti);
            if (resident || k >= kTrainSlots) continue;
            if (ensure_record(c, ti)) return TFG_ERR_CUDA;
            CK(cudaMemcpyAsync(c->d_stage_in + uint64_t(k) * rec_n, c->tiles[ti].rec, rec_n * sizeof(float),
                               cudaMemcpyHostToDevice, c->side));
            c->stage_tile[k++] = ti;
        }
        CK(cudaEventRecord(c->ev_stage_in, c->side));
    }
    CK(cudaStreamWaitEvent(c->side, c->ev_swap, 0));
    return stage_window(c, back, pr, pc, c->side);
}

TFG_API int tfg_window_tiles(tfg_ctx* c, int32_t* r4, int32_t* c4) {
    if (!c) return -1;
    for (int k = 0; k < c->nslots; ++k) {
        r4[k] = c->slot_tile[k] / c->cols;
        c4[k] = c->slot_tile[k] % c->cols;
    }
    return c->nslots;
}

TFG_API int tfg_accept_count(tfg_ctx* c, uint64_t* n) {
    if (!c) return fail(TFG_ERR_INVALID, "accept_count: null context");
    *n = c->nslots ? read_accept_count(c) : 0;
    return 0;
}

TFG_API int tfg_accept_export(tfg_ctx* c, uint64_t* out, uint64_t cap) {
    uint64_t n = std::min(cap, read_accept_count(c));
    CK(cudaMemcpyAsync(out, c->win[c->front].d_accept, n * 8, cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
    return 0;
}

// ---------------------------------------------------------------- training iteration
TFG_API int tfg_sample(tfg_ctx* c, uint64_t iter, uint64_t ray_begin, int n_rays, int jitter,
                       uint64_t* n_samples) {
    if (!c || c->nslots == 0) return fail(TFG_ERR_STATE, "sample: call set_window first");

    CK(cudaSetDevice(c->device));
    RaygenArgs a = base_raygen(c);
    a.accept = c->win[c->front].d_accept;
    a.n_accept_dev = c->win[c->front].d_n;
    a.memo_rays = c->win[c->front].d_mrays;
    a.iter = iter;
    a.ray_begin = ray_begin;
    a.n_rays = n_rays;
    a.jitter = jitter;
    c->render_mode = false;
    int rc = run_sampler(c, a);
    if (rc) return rc;
    if (n_samples) {
        rc = sync_status(c);
        if (rc) return rc;
        *n_samples = c->h_status->n_samples;
    }
    return 0;
}

TFG_API int tfg_sample_pixels(tfg_ctx* c, const int32_t* pixels, int n_rays, uint64_t* n_samples) {
    if (!c || c->nslots == 0) return fail(TFG_ERR_STATE, "sample_pixels: call set_window first");
    if (n_rays <= 0 || n_rays > c->max_rays) return fail(TFG_ERR_INVALID, "sample_pixels: n_rays");
    CK(cudaSetDevice(c->device));
    CK(cudaMemcpyAsync(c->d_pixels, pixels, size_t(n_rays) * 12, cudaMemcpyHostToDevice, c->st));
    RaygenArgs a = base_raygen(c);
    a.pixels = c->d_pixels;
    a.n_rays = n_rays;
    a.jitter = 0;
    c->render_mode = false;
    int rc = run_sampler(c, a);
    if (rc) return rc;
    rc = sync_status(c);
    if (rc) return rc;
    if (n_samples) *n_samples = c->h_status->n_samples;
    return 0;
}

TFG_API int tfg_forward_backward(tfg_ctx* c, uint64_t iter, uint64_t ray_begin, int n_rays) {
    int rc = tfg_sample(c, iter, ray_begin, n_rays, 1, nullptr);
    if (rc) return rc;
    if ((rc = run_forward(c, train_ptrs(c)))) return rc;
    if ((rc = run_composite(c, true))) return rc;
    return run_backward(c);
}

TFG_API int tfg_optimizer_step(tfg_ctx* c, uint64_t iter) {
    if (!c || c->nslots == 0) return fail(TFG_ERR_STATE, "optimizer_step: no window");
    CK(cudaSetDevice(c->device));
    const tfg_train_config& t = c->tc;
    auto lr_at = [&](double base, uint64_t step) {
        if (t.lr_decay_rate == 1.0) return base;
        return base * std::pow(t.lr_decay_rate, double(step) / double(t.lr_decay_steps));
    };
    AdamArgs a{};
    a.params = c->d_params;
    a.grads = c->d_grads;
    a.m = c->d_m;
    a.v = c->d_v;
    a.beta1 = t.beta1;
    a.beta2 = t.beta2;
    a.omb1 = 1.0f - t.beta1;
    a.omb2 = 1.0f - t.beta2;
    a.eps = t.eps;
    a.group_flags = c->d_group_flags;
    a.sticky = c->d_sticky;
    // bound the host's list of unverified steps (callers that never read the
    // status): settle it every 4096 steps
    if (c->unverified.size() >= 4096) {
        int rc = settle_steps(c);
        if (rc) return rc;
    }
    a.seq = ++c->step_seq;
    {
        tfg_ctx::StepRec r{};
        r.seq = a.seq;
        r.nslots = c->nslots;
        for (int k = 0; k < c->nslots; ++k) r.tile[k] = c->slot_tile[k];
        c->unverified.push_back(r);
    }
    a.enc16 = c->d_enc16;
    a.enc16_stride = c->enc16_stride;
    auto group = [&](AdamGroup& G, uint64_t off, uint64_t cnt, double base, uint64_t& step, int half_slot) {
        uint64_t s = ++step;
        G.offset = off;
        G.count = cnt;
        G.half_slot = half_slot;
        G.lr = float(lr_at(base, s));
        G.bc1 = float(1.0 - std::pow(double(t.beta1), double(s)));
        G.bc2 = float(1.0 - std::pow(double(t.beta2), double(s)));
    };
    int ng = 0;
    for (int k = 0; k < c->nslots; ++k) {
        TileHost& th = c->tiles[c->slot_tile[k]];
        group(a.g[ng++], uint64_t(k) * c->stride, c->enc_n, t.lr_field, th.enc_step, k);
        group(a.g[ng++], uint64_t(k) * c->stride + c->dn_off, c->dn_n, t.lr_field, th.dnet_step, -1);
    }
    group(a.g[ng++], c->color_off, c->n_params - c->color_off, t.lr_color, c->color_step, -1);
    a.n_groups = ng;
    // the colour group sits after the 4-slot region; a 1-slot window leaves a gap
    uint64_t total = c->n_params;
    CK(cudaMemsetAsync(c->d_group_flags, 0, 16 * 4, c->st));
    if (c->nslots < kTrainSlots) {
        // gap between slot region and colour: give it a zero-lr pseudo group
        for (int g = ng; g > 2 * c->nslots; --g) a.g[g] = a.g[g - 1];
        AdamGroup gap{};
        gap.half_slot = -1;
        gap.offset = uint64_t(c->nslots) * c->stride;
        gap.count = c->color_off - gap.offset;
        gap.lr = 0.f;
        gap.bc1 = gap.bc2 = 1.f;
        a.g[2 * c->nslots] = gap;
        a.n_groups = ng + 1;
    }
    for (int g = 0; g < a.n_groups; ++g)  // the Adam kernels stream float4s within one group
        if (a.g[g].offset % 4 != 0) return fail(TFG_ERR_INVALID, "optimizer_step: group offset not 4-aligned");
    {
        PhaseScope ps(c, kPhAdam);
        launch_adam(a, total, c->st, &c->launches);
    }
    CK(cudaGetLastError());
    int interval = c->fc.occupancy_interval;
    if (interval > 0 && (iter + 1) % uint64_t(interval) == 0) {
        uint64_t keys[kTrainSlots];
        for (int k = 0; k < c->nslots; ++k) {
            int ti = c->slot_tile[k];
            keys[k] = hash_combine(
                hash_combine(hash_combine(hash_combine(c->tc.seed, kPurposeOccupancy),
                                          uint64_t(ti / c->cols)),
                             uint64_t(ti % c->cols)),
                c->tiles[ti].dnet_step);
        }
        if (run_occupancy(c, true, keys)) return TFG_ERR_CUDA;
    }
    return 0;
}

TFG_API int tfg_read_loss(tfg_ctx* c, float* loss) {
    if (!c) return fail(TFG_ERR_INVALID, "read_loss: null context");
    int rc = sync_status(c);  // rolls back the step counts of skipped (non-finite) steps, once
    if (loss) *loss = float(c->h_status->loss / (3.0 * double(c->tc.batch_rays)));
    return rc;
}

// Pipelined status reads: request = an asynchronous snapshot of the loss /
// status of everything enqueued so far (pinned ring, one event each); poll =
// wait for the oldest snapshot and report it exactly as tfg_read_loss would
// (errors, non-finite rollback).  A training loop can request after step i
// and poll after enqueueing step i+1, so the host never drains the stream.
TFG_API int tfg_loss_request(tfg_ctx* c) {
    if (!c) return fail(TFG_ERR_INVALID, "loss_request: null context");
    if (c->ring_head - c->ring_tail >= uint32_t(tfg_ctx::kRing))
        return fail(TFG_ERR_STATE, "loss_request: 4 requests outstanding; poll first");
    CK(cudaSetDevice(c->device));
    if (!c->h_ring) {
        CK(cudaHostAlloc(reinterpret_cast<void**>(&c->h_ring), tfg_ctx::kRing * sizeof(Status), cudaHostAllocDefault));
        CK(cudaHostAlloc(reinterpret_cast<void**>(&c->h_ring_sticky), tfg_ctx::kRing * 16, cudaHostAllocDefault));
        for (auto& e : c->ev_ring) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    const uint32_t k = c->ring_head % tfg_ctx::kRing;
    CK(cudaMemcpyAsync(c->h_ring + k, c->d_status, sizeof(Status), cudaMemcpyDeviceToHost, c->st));
    CK(cudaMemcpyAsync(c->h_ring_sticky + 4 * k, c->d_sticky, 16, cudaMemcpyDeviceToHost, c->st));
    CK(cudaEventRecord(c->ev_ring[k], c->st));
    c->ring_seq[k] = c->step_seq;
    c->d2h_bytes += sizeof(Status) + 16;
    ++c->ring_head;
    return 0;
}

TFG_API int tfg_loss_poll(tfg_ctx* c, float* loss) {
    if (!c) return fail(TFG_ERR_INVALID, "loss_poll: null context");
    if (c->ring_head == c->ring_tail) return fail(TFG_ERR_STATE, "loss_poll: no outstanding loss_request");
    const uint32_t k = c->ring_tail % tfg_ctx::kRing;
    CK(cudaEventSynchronize(c->ev_ring[k]));
    ++c->ring_tail;
    *c->h_status = c->h_ring[k];
    consume_sticky(c, c->h_ring_sticky + 4 * k, c->ring_seq[k]);
    if (loss) *loss = float(c->h_status->loss / (3.0 * double(c->tc.batch_rays)));
    return check_status(c);
}

TFG_API int tfg_train_step(tfg_ctx* c, uint64_t iter, uint64_t ray_begin, int n_rays,
                           float* loss) {
    int rc = tfg_forward_backward(c, iter, ray_begin, n_rays);
    if (rc) return rc;
    rc = tfg_optimizer_step(c, iter);
    if (rc) return rc;
    return tfg_read_loss(c, loss);
}

TFG_API int tfg_grad_buffer(tfg_ctx* c, void** dptr, uint64_t* count) {
    if (!c) return fail(TFG_ERR_INVALID, "grad_buffer: null context");
    *dptr = c->d_grads;
    *count = c->n_params;
    return 0;
}

// ---------------------------------------------------------------- parity surface
TFG_API int tfg_batch_export(tfg_ctx* c, tfg_batch_view* out) {
    if (!c || !c->have_batch) return fail(TFG_ERR_STATE, "batch_export: no batch");
    HostBatch hb;
    int rc = fetch_batch_meta(c, hb);
    if (rc) return rc;
    uint64_t S = hb.n_samples;
    if (out->capacity < S) return fail(TFG_ERR_INVALID, "batch_export: capacity too small");
    std::unique_ptr<float4[]> loc;
    std::unique_ptr<float2[]> td;
    std::unique_ptr<uint8_t[]> ep;
    if ((rc = pull_samples(hb, c->s.local, loc)) || (rc = pull_samples(hb, c->s.td, td)) ||
        (rc = pull_samples(hb, c->s.endpoint, ep)))
        return rc;
    int n = c->cur_rays;
    std::vector<uint32_t> cnt(n, 0);
    for (int i = 0; i < n; ++i) {
        const RayRec& R = hb.rays[i];
        if (out->rays) {
            tfg_ray_entry& e = out->rays[i];
            for (int k = 0; k < 3; ++k) {
                e.origin[k] = R.o[k];
                e.direction[k] = R.d[k];
                e.target[k] = R.target[k];
            }
            e.image_id = R.view;
            e.row = R.row;
            e.col = R.col;
        }
        if (R.status == 0)
            for (int k = 0; k < R.nseg; ++k) cnt[i] += R.cnt[k];
    }
    if (out->offsets) {
        out->offsets[0] = 0;
        for (int i = 0; i < n; ++i) out->offsets[i + 1] = out->offsets[i] + cnt[i];
    }
    for_samples(c, hb, [&](int, uint64_t q, uint64_t pos, int slot) {
        if (out->t) out->t[q] = td[pos].x;
        if (out->delta) out->delta[q] = td[pos].y;
        if (out->local) {
            out->local[3 * q] = loc[pos].x;
            out->local[3 * q + 1] = loc[pos].y;
            out->local[3 * q + 2] = loc[pos].z;
        }
        if (out->slot) out->slot[q] = uint8_t(slot);
        if (out->endpoint) out->endpoint[q] = ep[pos];
    });
    return 0;
}

// A caller-built RaySegmentBatch (ray_batch.hpp:13-49) becomes the context's
// current batch: the forward_batch / backward_batch drop-in (field.hpp:186-197).
TFG_API int tfg_batch_import(tfg_ctx* c, const tfg_batch_view* in, int n_rays) {
    if (!c || !in) return fail(TFG_ERR_INVALID, "batch_import: null argument");
    if (c->nslots == 0) return fail(TFG_ERR_STATE, "batch_import: no loaded slots (set_window or set_slot_params)");
    if (n_rays <= 0 || n_rays > c->max_rays) return fail(TFG_ERR_INVALID, "batch_import: n_rays outside (0, max_rays]");
    if (!in->rays || !in->offsets || !in->t || !in->delta || !in->local || !in->slot || !in->endpoint)
        return fail(TFG_ERR_INVALID, "batch_import: every batch array is required");
    if (in->offsets[0] != 0) return fail(TFG_ERR_INVALID, "batch_import: offsets[0] must be 0");
    for (int i = 0; i < n_rays; ++i)
        if (in->offsets[i + 1] < in->offsets[i]) return fail(TFG_ERR_INVALID, "batch_import: offsets must ascend");
    const uint64_t S = in->offsets[n_rays];
    if (S > c->sample_cap) return fail(TFG_ERR_INVALID, "batch_import: batch exceeds the sample capacity of the context");
    CK(cudaSetDevice(c->device));
    // staging: rays | offsets | t | delta | local | slot | endpoint
    const uint64_t cap = c->sample_cap, mr = uint64_t(c->max_rays);
    const uint64_t o_off = mr * sizeof(tfg_ray_entry), o_t = o_off + ((mr + 1) * 4 + 15) / 16 * 16,
                   o_de = o_t + cap * 4, o_lo = o_de + cap * 4, o_sl = o_lo + cap * 12, o_ep = o_sl + cap,
                   total = o_ep + cap;
    if (!c->d_imp && dalloc(c, &c->d_imp, total)) return TFG_ERR_CUDA;
    uint8_t* b = c->d_imp;
    CK(cudaMemcpyAsync(b, in->rays, size_t(n_rays) * sizeof(tfg_ray_entry), cudaMemcpyHostToDevice, c->st));
    CK(cudaMemcpyAsync(b + o_off, in->offsets, size_t(n_rays + 1) * 4, cudaMemcpyHostToDevice, c->st));
    CK(cudaMemcpyAsync(b + o_t, in->t, S * 4, cudaMemcpyHostToDevice, c->st));
    CK(cudaMemcpyAsync(b + o_de, in->delta, S * 4, cudaMemcpyHostToDevice, c->st));
    CK(cudaMemcpyAsync(b + o_lo, in->local, S * 12, cudaMemcpyHostToDevice, c->st));
    CK(cudaMemcpyAsync(b + o_sl, in->slot, S, cudaMemcpyHostToDevice, c->st));
    CK(cudaMemcpyAsync(b + o_ep, in->endpoint, S, cudaMemcpyHostToDevice, c->st));
    c->h2d_bytes += n_rays * (sizeof(tfg_ray_entry) + 4) + S * 22;
    ImportArgs a{};
    a.rays = reinterpret_cast<const tfg_ray_entry*>(b);
    a.offsets = reinterpret_cast<const uint32_t*>(b + o_off);
    a.t = reinterpret_cast<const float*>(b + o_t);
    a.delta = reinterpret_cast<const float*>(b + o_de);
    a.local = reinterpret_cast<const float*>(b + o_lo);
    a.slot = b + o_sl;
    a.endpoint = b + o_ep;
    a.n_rays = n_rays;
    a.nslots = c->nslots;
    {
        PhaseScope ps(c, kPhSampler);
        CK(cudaMemsetAsync(c->d_status, 0, sizeof(Status), c->st));
        if (launch_import(a, c->d_rays, c->d_hdr, c->d_venc, c->d_counts, c->d_P, c->d_block_sums, c->d_tiles, c->max_tiles,
                          c->s, c->sample_cap, c->d_status, c->st, &c->launches))
            return fail(TFG_ERR_INVALID, "batch_import: scan capacity exceeded");
        CK(cudaGetLastError());
    }
    c->cur_rays = n_rays;
    c->have_batch = true;
    c->fwd_done = false;
    c->io_fwd = false;
    c->render_mode = false;
    return sync_status(c);
}

// Loads caller-owned parameters into a slot (FieldParamView, field.hpp:130-137)
// or the colour net (ColorParamView, :139-144).  With no window set, slots
// are bound detached (no tile record): forward/backward only.
TFG_API int tfg_set_slot_params(tfg_ctx* c, int slot, const float* enc, const float* dnet) {
    if (!c || slot < 0 || slot >= kTrainSlots) return fail(TFG_ERR_INVALID, "set_slot_params: bad slot");
    CK(cudaSetDevice(c->device));
    if (slot >= c->nslots) {
        if (c->pos_r >= 0) return fail(TFG_ERR_INVALID, "set_slot_params: slot outside the window");
        for (int k = c->nslots; k <= slot; ++k) c->slot_tile[k] = -1;
        c->nslots = slot + 1;
        c->slots.n = c->nslots;  // batch layout [slot][ray] of imported batches
    }
    CK(cudaStreamSynchronize(c->st));
    const uint64_t off = uint64_t(slot) * c->stride;
    if (enc) CK(cudaMemcpy(c->d_params + off, enc, c->enc_n * 4, cudaMemcpyHostToDevice));
    if (dnet) CK(cudaMemcpy(c->d_params + off + c->dn_off, dnet, (c->dn_n) * 4, cudaMemcpyHostToDevice));
    c->fwd_done = false;
    c->enc16_dirty = true;
    return 0;
}

TFG_API int tfg_set_color_params(tfg_ctx* c, const float* params) {
    if (!c || !params) return fail(TFG_ERR_INVALID, "set_color_params: null argument");
    CK(cudaSetDevice(c->device));
    CK(cudaStreamSynchronize(c->st));
    CK(cudaMemcpy(c->d_params + c->color_off, params, (c->n_params - c->color_off) * 4, cudaMemcpyHostToDevice));
    c->fwd_done = false;
    return 0;
}

// Writes caller-given per-sample sigma / rgb (ray order) into the batch's
// field outputs: compositing (render + loss + render backward) then runs on
// exactly these values.
TFG_API int tfg_set_field_outputs(tfg_ctx* c, const float* sigma, const float* rgb) {
    if (!c || !c->have_batch) return fail(TFG_ERR_STATE, "set_field_outputs: no batch");
    if (!sigma || !rgb) return fail(TFG_ERR_INVALID, "set_field_outputs: null argument");
    HostBatch hb;
    int rc = fetch_batch_meta(c, hb);
    if (rc) return rc;
    std::unique_ptr<float4[]> io(new float4[std::max<uint64_t>(1, hb.extent)]);
    for_samples(c, hb, [&](int, uint64_t q, uint64_t pos, int) {
        io[pos] = make_float4(sigma[q], rgb[3 * q], rgb[3 * q + 1], rgb[3 * q + 2]);
    });
    if ((rc = push_samples(hb, io.get(), c->s.io))) return rc;
    c->io_fwd = true;
    return 0;
}

// backward_batch from caller-given d_sigma / d_rgb (ray order; gradients with
// respect to the field outputs, field.hpp:193-197): converted to the
// pre-activation gradients K4 consumes (density_activation / sigmoid
// derivatives, nn.hpp:270-285) against the forward's sigma / rgb, then the
// field backward into the flat gradient buffer (zeroed first).
TFG_API int tfg_field_backward_from(tfg_ctx* c, const float* d_sigma, const float* d_rgb) {
    if (!c || !c->have_batch) return fail(TFG_ERR_STATE, "field_backward_from: no batch");
    if (!d_sigma || !d_rgb) return fail(TFG_ERR_INVALID, "field_backward_from: null argument");
    if (!c->fwd_done || !c->io_fwd)
        return fail(TFG_ERR_STATE, "field_backward_from: run field_forward on this batch first");
    HostBatch hb;
    int rc = fetch_batch_meta(c, hb);
    if (rc) return rc;
    std::unique_ptr<float4[]> io;
    if ((rc = pull_samples(hb, c->s.io, io))) return rc;
    const float dmax = c->fc.density_max;
    for_samples(c, hb, [&](int, uint64_t q, uint64_t pos, int) {
        const float4 f = io[pos];
        const float dr = d_rgb[3 * q], dg = d_rgb[3 * q + 1], db = d_rgb[3 * q + 2];
        io[pos] = make_float4(f.x >= dmax ? 0.f : d_sigma[q] * f.x, dr * f.y * (1.f - f.y), dg * f.z * (1.f - f.z),
                              db * f.w * (1.f - f.w));
    });
    if ((rc = push_samples(hb, io.get(), c->s.io))) return rc;
    c->io_fwd = false;
    if ((rc = run_backward(c))) return rc;
    CK(cudaStreamSynchronize(c->st));
    return 0;
}

// adam_step (field.hpp:45-48) over caller spans (host or device memory):
// state = (m, v, *step), schedule = (lr_base, lr_decay_rate, lr_decay_steps),
// config = (beta1, beta2, eps).  Non-finite gradients: TFG_ERR_NONFINITE
// naming `group`, nothing updated, step unchanged.  Synchronous.
TFG_API int tfg_adam_step(tfg_ctx* c, float* params, const float* grads, float* m, float* v, uint64_t n,
                          uint64_t* step, double lr_base, double lr_decay_rate, uint64_t lr_decay_steps,
                          float beta1, float beta2, float eps, const char* group) {
    if (!c || !params || !grads || !m || !v || !step) return fail(TFG_ERR_INVALID, "adam_step: null argument");
    if (n == 0) {
        ++*step;
        return 0;
    }
    CK(cudaSetDevice(c->device));
    auto on_device = [](const void* p) {
        cudaPointerAttributes at{};
        if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
            cudaGetLastError();
            return false;
        }
        return (at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged) &&
               (reinterpret_cast<uintptr_t>(p) & 15) == 0;
    };
    const bool dev = on_device(params) && on_device(grads) && on_device(m) && on_device(v);
    float *dp = params, *dm = m, *dv = v;
    const float* dg = grads;
    void* scratch = nullptr;
    uint32_t* flags = nullptr;
    CK(cudaMallocAsync(reinterpret_cast<void**>(&flags), 32 * 4, c->st));
    CK(cudaMemsetAsync(flags, 0, 32 * 4, c->st));
    if (!dev) {
        const size_t nb = (n * 4 + 255) / 256 * 256;
        CK(cudaMallocAsync(&scratch, 4 * nb, c->st));
        dp = static_cast<float*>(scratch);
        float* g = reinterpret_cast<float*>(static_cast<char*>(scratch) + nb);
        dm = reinterpret_cast<float*>(static_cast<char*>(scratch) + 2 * nb);
        dv = reinterpret_cast<float*>(static_cast<char*>(scratch) + 3 * nb);
        CK(cudaMemcpyAsync(dp, params, n * 4, cudaMemcpyDefault, c->st));
        CK(cudaMemcpyAsync(g, grads, n * 4, cudaMemcpyDefault, c->st));
        CK(cudaMemcpyAsync(dm, m, n * 4, cudaMemcpyDefault, c->st));
        CK(cudaMemcpyAsync(dv, v, n * 4, cudaMemcpyDefault, c->st));
        dg = g;
    }
    const uint64_t s = *step + 1;
    AdamArgs a{};
    a.params = dp;
    a.grads = dg;
    a.m = dm;
    a.v = dv;
    a.beta1 = beta1;
    a.beta2 = beta2;
    a.omb1 = 1.0f - beta1;
    a.omb2 = 1.0f - beta2;
    a.eps = eps;
    a.group_flags = flags;
    a.sticky = flags + 16;
    a.seq = 1;
    a.n_groups = 1;
    a.g[0].offset = 0;
    a.g[0].count = n;
    a.g[0].half_slot = -1;
    a.g[0].lr = float(lr_decay_rate == 1.0 ? lr_base
                                           : lr_base * std::pow(lr_decay_rate, double(s) / double(lr_decay_steps)));
    a.g[0].bc1 = float(1.0 - std::pow(double(beta1), double(s)));
    a.g[0].bc2 = float(1.0 - std::pow(double(beta2), double(s)));
    launch_adam(a, n, c->st, &c->launches);
    CK(cudaGetLastError());
    uint32_t bad = 0;
    CK(cudaMemcpyAsync(&bad, flags + 16, 4, cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
    if (!dev && bad == 0) {  // staged: the update goes back to the caller's spans
        CK(cudaMemcpyAsync(params, dp, n * 4, cudaMemcpyDefault, c->st));
        CK(cudaMemcpyAsync(m, dm, n * 4, cudaMemcpyDefault, c->st));
        CK(cudaMemcpyAsync(v, dv, n * 4, cudaMemcpyDefault, c->st));
    }
    if (scratch) CK(cudaFreeAsync(scratch, c->st));
    CK(cudaFreeAsync(flags, c->st));
    CK(cudaStreamSynchronize(c->st));
    if (bad) return fail(TFG_ERR_NONFINITE, std::string("adam_step: non-finite gradient in group ") + (group ? group : "?"));
    ++*step;
    return 0;
}

TFG_API int tfg_field_forward(tfg_ctx* c, float* sigma, float* rgb) {
    if (!c || !c->have_batch) return fail(TFG_ERR_STATE, "field_forward: no batch");
    int rc = run_forward(c, train_ptrs(c));
    if (rc) return rc;
    if (!sigma && !rgb) return 0;
    HostBatch hb;
    if ((rc = fetch_batch_meta(c, hb))) return rc;
    std::unique_ptr<float4[]> io;
    if ((rc = pull_samples(hb, c->s.io, io))) return rc;
    for_samples(c, hb, [&](int, uint64_t q, uint64_t pos, int) {
        if (sigma) sigma[q] = io[pos].x;
        if (rgb) {
            rgb[3 * q] = io[pos].y;
            rgb[3 * q + 1] = io[pos].z;
            rgb[3 * q + 2] = io[pos].w;
        }
    });
    return 0;
}

TFG_API int tfg_composite(tfg_ctx* c, float* ray_rgb, float* ray_depth, float* ray_opacity,
                          float* d_sigma, float* d_rgb, float* loss) {
    if (!c || !c->have_batch) return fail(TFG_ERR_STATE, "composite: no batch");
    if (!c->d_export && dalloc(c, &c->d_export, c->sample_cap)) return TFG_ERR_CUDA;
    int rc = run_composite(c, true, c->d_export);
    if (rc) return rc;
    HostBatch hb;
    if ((rc = fetch_batch_meta(c, hb))) return rc;
    int n = c->cur_rays;
    std::vector<float> ro(5 * uint64_t(c->max_rays));
    CK(cudaMemcpy(ro.data(), c->d_ray_out, ro.size() * 4, cudaMemcpyDeviceToHost));
    for (int i = 0; i < n; ++i) {
        if (ray_rgb)
            for (int k = 0; k < 3; ++k) ray_rgb[3 * i + k] = ro[3 * i + k];
        if (ray_depth) ray_depth[i] = ro[3 * uint64_t(c->max_rays) + i];
        if (ray_opacity) ray_opacity[i] = ro[4 * uint64_t(c->max_rays) + i];
    }
    if (d_sigma || d_rgb) {
        std::unique_ptr<float4[]> io;
        if ((rc = pull_samples(hb, c->d_export, io))) return rc;
        for_samples(c, hb, [&](int, uint64_t q, uint64_t pos, int) {
            if (d_sigma) d_sigma[q] = io[pos].x;
            if (d_rgb) {
                d_rgb[3 * q] = io[pos].y;
                d_rgb[3 * q + 1] = io[pos].z;
                d_rgb[3 * q + 2] = io[pos].w;
            }
        });
    }
    if (loss) *loss = float(c->h_status->loss / (3.0 * double(c->tc.batch_rays)));
    return 0;
}

TFG_API int tfg_field_backward(tfg_ctx* c) {
    if (!c || !c->have_batch) return fail(TFG_ERR_STATE, "field_backward: no batch");
    int rc = run_backward(c);
    if (rc) return rc;
    CK(cudaStreamSynchronize(c->st));
    return 0;
}

TFG_API int tfg_get_grads(tfg_ctx* c, int slot, float* enc, float* dnet, float* color) {
    if (!c || slot < 0 || slot >= c->nslots) return fail(TFG_ERR_INVALID, "get_grads: bad slot");
    CK(cudaStreamSynchronize(c->st));
    uint64_t off = uint64_t(slot) * c->stride;
    if (enc) CK(cudaMemcpy(enc, c->d_grads + off, c->enc_n * 4, cudaMemcpyDeviceToHost));
    if (dnet)
        CK(cudaMemcpy(dnet, c->d_grads + off + c->dn_off, (c->dn_n) * 4,
                      cudaMemcpyDeviceToHost));
    if (color)
        CK(cudaMemcpy(color, c->d_grads + c->color_off, (c->n_params - c->color_off) * 4,
                      cudaMemcpyDeviceToHost));
    return 0;
}

TFG_API int tfg_get_tile_state(tfg_ctx* c, int slot, tfg_tile_state* o) {
    if (!c || slot < 0 || slot >= c->nslots) return fail(TFG_ERR_INVALID, "get_tile_state: bad slot");
    if (settle_steps(c)) return TFG_ERR_CUDA;  // step counts of skipped steps rolled back
    CK(cudaStreamSynchronize(c->side));
    uint64_t off = uint64_t(slot) * c->stride;
    uint64_t dn = c->dn_n;
    auto cp = [&](float* dst, const float* src, uint64_t n) -> int {
        if (dst) CK(cudaMemcpy(dst, src, n * 4, cudaMemcpyDeviceToHost));
        return 0;
    };
    int rc = cp(o->enc, c->d_params + off, c->enc_n) | cp(o->dnet, c->d_params + off + c->dn_off, dn) |
             cp(o->enc_m, c->d_m + off, c->enc_n) | cp(o->enc_v, c->d_v + off, c->enc_n) |
             cp(o->dnet_m, c->d_m + off + c->dn_off, dn) | cp(o->dnet_v, c->d_v + off + c->dn_off, dn) |
             cp(o->occupancy, c->d_ema + uint64_t(slot) * kOccVox, kOccVox);
    const TileHost& th = c->tiles[c->slot_tile[slot]];
    o->enc_step = th.enc_step;
    o->dnet_step = th.dnet_step;
    return rc;
}

TFG_API int tfg_set_tile_state(tfg_ctx* c, int slot, const tfg_tile_state* in) {
    if (!c || slot < 0 || slot >= c->nslots) return fail(TFG_ERR_INVALID, "set_tile_state: bad slot");
    CK(cudaStreamSynchronize(c->st));
    uint64_t off = uint64_t(slot) * c->stride;
    uint64_t dn = c->dn_n;
    auto cp = [&](float* dst, const float* src, uint64_t n) -> int {
        if (src) CK(cudaMemcpy(dst, src, n * 4, cudaMemcpyHostToDevice));
        return 0;
    };
    int rc = cp(c->d_params + off, in->enc, c->enc_n) | cp(c->d_params + off + c->dn_off, in->dnet, dn) |
             cp(c->d_m + off, in->enc_m, c->enc_n) | cp(c->d_v + off, in->enc_v, c->enc_n) |
             cp(c->d_m + off + c->dn_off, in->dnet_m, dn) | cp(c->d_v + off + c->dn_off, in->dnet_v, dn) |
             cp(c->d_ema + uint64_t(slot) * kOccVox, in->occupancy, kOccVox);
    TileHost& th = c->tiles[c->slot_tile[slot]];
    th.enc_step = in->enc_step;
    th.dnet_step = in->dnet_step;
    c->enc16_dirty = true;
    if (rc) return rc;
    return run_occupancy(c, false, nullptr);
}

TFG_API int tfg_get_color(tfg_ctx* c, float* p, float* m, float* v, uint64_t* step) {
    if (!c) return fail(TFG_ERR_INVALID, "get_color: null context");
    if (settle_steps(c)) return TFG_ERR_CUDA;
    uint64_t n = c->n_params - c->color_off;
    if (p) CK(cudaMemcpy(p, c->d_params + c->color_off, n * 4, cudaMemcpyDeviceToHost));
    if (m) CK(cudaMemcpy(m, c->d_m + c->color_off, n * 4, cudaMemcpyDeviceToHost));
    if (v) CK(cudaMemcpy(v, c->d_v + c->color_off, n * 4, cudaMemcpyDeviceToHost));
    if (step) *step = c->color_step;
    return 0;
}

TFG_API int tfg_set_color(tfg_ctx* c, const float* p, const float* m, const float* v,
                          uint64_t step) {
    CK(cudaStreamSynchronize(c->st));
    uint64_t n = c->n_params - c->color_off;
    if (p) CK(cudaMemcpy(c->d_params + c->color_off, p, n * 4, cudaMemcpyHostToDevice));
    if (m) CK(cudaMemcpy(c->d_m + c->color_off, m, n * 4, cudaMemcpyHostToDevice));
    if (v) CK(cudaMemcpy(c->d_v + c->color_off, v, n * 4, cudaMemcpyHostToDevice));
    c->color_step = step;
    return 0;
}

TFG_API int tfg_update_occupancy(tfg_ctx* c) {
    if (!c || c->nslots == 0) return fail(TFG_ERR_STATE, "update_occupancy: no window");
    uint64_t keys[kTrainSlots];
    for (int k = 0; k < c->nslots; ++k) {
        int ti = c->slot_tile[k];
        keys[k] = hash_combine(hash_combine(hash_combine(hash_combine(c->tc.seed, kPurposeOccupancy),
                                                         uint64_t(ti / c->cols)),
                                            uint64_t(ti % c->cols)),
                               c->tiles[ti].dnet_step);
    }
    int rc = run_occupancy(c, true, keys);
    if (rc) return rc;
    CK(cudaStreamSynchronize(c->st));
    return 0;
}

TFG_API int tfg_get_memory_report(tfg_ctx* c, tfg_memory_report* o) {
    if (!c) return fail(TFG_ERR_INVALID, "memory_report: null context");
    std::memset(o, 0, sizeof(*o));
    o->tile_params = kTrainSlots * c->stride * 4;
    o->optimizer_moments = 2 * kTrainSlots * c->stride * 4 + kTrainSlots * c->stride * 4;  // m, v, grads
    o->occupancy = uint64_t(kTrainSlots) * kOccVox * 4 + uint64_t(kMaxSlots) * kOccWords * 4;
    o->crops = 2 * c->crop_cap;
    // accepted lists + the two window pixel memos + the build scratch
    o->accept_list = 2 * c->accept_cap * 8 + 2 * c->cand_cap * (4 + 48) + c->cand_cap * 8;
    o->batch_buffers = uint64_t(c->max_rays) * (sizeof(RayRec) + sizeof(RayHdr) + 96 + 8 * kMaxSlots + 20 + 12) +
                       c->sample_cap * (16 + 8 + 1 + 16);
    o->color_net = (c->n_params - c->color_off) * 4;
    o->total_device = c->bytes_total;
    return 0;
}

// ---------------------------------------------------------------- render path
TFG_API int tfg_render_setup(tfg_ctx* c, const int32_t* rows, const int32_t* cols, int n,
                             const tfg_tile_state* states, const float* color_params) {
    if (!c || c->n_views == 0) return fail(TFG_ERR_STATE, "render_setup: call set_scene first");
    if (n <= 0 || n > kMaxSlots) return fail(TFG_ERR_INVALID, "render_setup: 1..16 tiles");
    CK(cudaSetDevice(c->device));
    if (!c->d_rparams) {
        if (dalloc(c, &c->d_rparams, uint64_t(kMaxSlots) * c->stride)) return TFG_ERR_CUDA;
        if (dalloc(c, &c->d_rbits, uint64_t(kMaxSlots) * kOccWords)) return TFG_ERR_CUDA;
        if (dalloc(c, &c->d_rcolor, c->n_params - c->color_off)) return TFG_ERR_CUDA;
    }
    c->rn = n;
    c->rslots.n = n;
    std::vector<uint32_t> bits(kOccWords);
    for (int k = 0; k < n; ++k) {
        int ti = rows[k] * c->cols + cols[k];
        double b[6];
        tile_box(c, ti, b);
        for (int q = 0; q < 6; ++q) c->rslots.box[k][q] = b[q];
        for (int q = 0; q < 3; ++q) {
            c->rslots.frame[k][q] = b[q];
            c->rslots.frame[k][3 + q] = 1.0 / (b[3 + q] - b[q]);
        }
        float* dst = c->d_rparams + uint64_t(k) * c->stride;
        CK(cudaMemcpy(dst, states[k].enc, c->enc_n * 4, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(dst + c->dn_off, states[k].dnet, (c->dn_n) * 4, cudaMemcpyHostToDevice));
        for (int w = 0; w < kOccWords; ++w) {
            uint32_t word = 0;
            for (int q = 0; q < 32; ++q) {
                float e = states[k].occupancy ? states[k].occupancy[32 * w + q] : 1.0f;
                word |= (e >= c->fc.occupancy_threshold ? 1u : 0u) << q;
            }
            bits[w] = word;
        }
        CK(cudaMemcpy(c->d_rbits + uint64_t(k) * kOccWords, bits.data(), kOccWords * 4,
                      cudaMemcpyHostToDevice));
    }
    CK(cudaMemcpy(c->d_rcolor, color_params, (c->n_params - c->color_off) * 4, cudaMemcpyHostToDevice));
    // the render tiles' fp16 table shadows (after the training slots')
    launch_enc_half(c->d_rparams, c->stride, n, c->enc_n, c->enc16_stride,
                    static_cast<uint16_t*>(c->d_enc16) + uint64_t(kTrainSlots) * c->enc16_stride, c->st, &c->launches);
    CK(cudaStreamSynchronize(c->st));
    return 0;
}

// Forward-only path (cmd_render): midpoint samples over the
// render tiles, K2 forward, K3 forward; chunks of max_rays rays.
TFG_API int tfg_render_pixels(tfg_ctx* c, const tfg_rpc* cam, const int32_t* pixels, int n_rays,
                              float* rgb, float* depth, float* opacity) {
    if (!c || c->rn == 0) return fail(TFG_ERR_STATE, "render_pixels: call render_setup first");
    CK(cudaSetDevice(c->device));
    CK(cudaMemcpyAsync(c->d_rcam, cam, sizeof(tfg_rpc), cudaMemcpyHostToDevice, c->st));
    launch_loc_start(c->d_rcam, 1, c->roi.z_min, c->roi.z_max, c->d_rloc, c->st);
    FieldPtrs f{};
    for (int k = 0; k < c->rn; ++k) {
        f.enc[k] = c->d_rparams + uint64_t(k) * c->stride;
        f.enc16[k] = static_cast<uint16_t*>(c->d_enc16) + uint64_t(kTrainSlots + k) * c->enc16_stride;
        f.dnet[k] = f.enc[k] + c->dn_off;
        f.occ_bits[k] = c->d_rbits + uint64_t(k) * kOccWords;
    }
    f.color = c->d_rcolor;
    // Chunks of max_rays rays, software-pipelined: while the GPU renders chunk
    // i, the host stages chunk i+1's pixels into one pinned buffer and copies
    // chunk i-1's outputs out of the other; the GPU side copies only pinned
    // memory.
    const uint64_t M = uint64_t(c->max_rays);
    if (!c->h_rpix) {
        CK(cudaHostAlloc(reinterpret_cast<void**>(&c->h_rpix), 2 * M * 8, cudaHostAllocDefault));
        CK(cudaHostAlloc(reinterpret_cast<void**>(&c->h_rout), 2 * M * 20, cudaHostAllocDefault));
        CK(cudaHostAlloc(reinterpret_cast<void**>(&c->h_rstat), 2 * sizeof(Status), cudaHostAllocDefault));
        for (auto& e : c->ev_rdone) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    const int nch = int((uint64_t(n_rays) + M - 1) / M);
    auto chunk_n = [&](int i) { return int(std::min<uint64_t>(M, uint64_t(n_rays) - uint64_t(i) * M)); };
    auto stage_in = [&](int i) {
        std::memcpy(c->h_rpix + (i & 1) * 2 * M, pixels + 2 * uint64_t(i) * M, size_t(chunk_n(i)) * 8);
    };
    auto drain = [&](int i) -> int {
        CK(cudaEventSynchronize(c->ev_rdone[i & 1]));
        const Status& st = c->h_rstat[i & 1];
        if (st.bits & (kStatusSampleOverflow | kStatusSegOverflow)) {
            *c->h_status = st;
            return check_status(c);
        }
        const float* ro = c->h_rout + (i & 1) * 5 * M;
        uint64_t b0 = uint64_t(i) * M, nb = uint64_t(chunk_n(i));
        if (rgb) std::memcpy(rgb + 3 * b0, ro, nb * 12);
        if (depth) std::memcpy(depth + b0, ro + 3 * M, nb * 4);
        if (opacity) std::memcpy(opacity + b0, ro + 4 * M, nb * 4);
        return 0;
    };
    // a previous call that stopped on an error may still have copies queued
    // from the pinned buffers
    CK(cudaStreamSynchronize(c->st));
    if (nch > 0) stage_in(0);
    int drained = 0;  // chunks [0, drained) are copied out
    for (int i = 0; i < nch; ++i) {
        const int b = i & 1, nb = chunk_n(i);
        CK(cudaMemcpyAsync(c->d_pixels, c->h_rpix + b * 2 * M, size_t(nb) * 8, cudaMemcpyHostToDevice, c->st));
        RaygenArgs a{};
        a.cams = c->d_rcam;
        a.loc = c->d_rloc;
        a.pixels = c->d_pixels;
        a.pixel_pairs = 1;
        a.n_rays = nb;
        a.z_min = c->roi.z_min;
        a.z_max = c->roi.z_max;
        a.spm = c->tc.samples_per_meter;
        a.cap = c->tc.max_samples_per_ray;
        a.delta_cap = c->tc.delta_cap;
        a.slots = c->rslots;
        for (int k = 0; k < c->rn; ++k) a.occ_bits[k] = f.occ_bits[k];
        int rc = run_sampler(c, a);
        if (rc) return rc;
        c->render_mode = true;
        if ((rc = run_forward(c, f))) return rc;
        c->fwd_done = false;
        if ((rc = run_composite(c, false))) return rc;
        float* ho = c->h_rout + b * 5 * M;
        CK(cudaMemcpyAsync(ho, c->d_ray_out, size_t(nb) * 12, cudaMemcpyDeviceToHost, c->st));
        CK(cudaMemcpyAsync(ho + 3 * M, c->d_ray_out + 3 * M, size_t(nb) * 4, cudaMemcpyDeviceToHost, c->st));
        CK(cudaMemcpyAsync(ho + 4 * M, c->d_ray_out + 4 * M, size_t(nb) * 4, cudaMemcpyDeviceToHost, c->st));
        CK(cudaMemcpyAsync(c->h_rstat + b, c->d_status, sizeof(Status), cudaMemcpyDeviceToHost, c->st));
        CK(cudaEventRecord(c->ev_rdone[b], c->st));
        c->d2h_bytes += uint64_t(nb) * 20 + sizeof(Status);
        if (i + 1 < nch) {
            // chunk i-1 used the buffers chunk i+1 is about to take
            if (i >= 1 && (rc = drain(i - 1))) return rc;
            drained = i;
            stage_in(i + 1);
        }
    }
    for (int i = drained; i < nch; ++i) {
        int rc = drain(i);
        if (rc) return rc;
    }
    c->have_batch = false;
    return 0;
}

// ---------------------------------------------------------------- instrumentation
TFG_API int tfg_kernel_launch_count(tfg_ctx* c, uint64_t* n) {
    if (!c) return fail(TFG_ERR_INVALID, "kernel_launch_count: null context");
    *n = c->launches;
    return 0;
}

TFG_API int tfg_profile_enable(tfg_ctx* c, int on) {
    if (!c) return fail(TFG_ERR_INVALID, "profile_enable: null context");
    prof_collect(c);
    c->prof = on != 0;
    for (int p = 0; p < kNumPhases; ++p) {
        c->prof_ms[p] = 0;
        c->prof_n[p] = 0;
        c->prof_launch[p] = 0;
    }
    return 0;
}

// Accumulated device ms, bracket counts and kernel launches per phase since
// the last tfg_profile_enable (synchronises on the recorded events).
TFG_API int tfg_profile_read(tfg_ctx* c, const char** names, double* ms, uint64_t* launches,
                             int capacity, int* n_out) {
    if (!c) return fail(TFG_ERR_INVALID, "profile_read: null context");
    prof_collect(c);
    int n = std::min(capacity, int(kNumPhases));
    for (int p = 0; p < n; ++p) {
        if (names) names[p] = kPhaseNames[p];
        if (ms) ms[p] = c->prof_ms[p];
        if (launches) launches[p] = c->prof_launch[p];
    }
    if (n_out) *n_out = n;
    return 0;
}

TFG_API int tfg_last_batch(tfg_ctx* c, int* n_rays, uint64_t* n_samples) {
    if (!c) return fail(TFG_ERR_INVALID, "last_batch: null context");
    int rc = sync_status(c);
    if (n_rays) *n_rays = c->cur_rays;
    if (n_samples) *n_samples = c->h_status->n_samples;
    return rc;
}

// TileField::create (field.hpp:93) on the host into caller buffers (enc, dnet,
// occupancy all 1.0; moments zero when given).
TFG_API int tfg_tile_init(const tfg_field_config* fc, uint64_t seed, int row, int col,
                          tfg_tile_state* o) {
    uint64_t enc, dn;
    tfg_param_counts(fc, &enc, &dn, nullptr);
    Rng re(hash_combine(hash_combine(hash_combine(seed, kPurposeTileEnc), uint64_t(row)), uint64_t(col)));
    if (o->enc)
        for (uint64_t i = 0; i < enc; ++i) o->enc[i] = float(re.uniform(-1e-4, 1e-4));
    Rng rd(hash_combine(hash_combine(hash_combine(seed, kPurposeTileDnet), uint64_t(row)), uint64_t(col)));
    const int dw[3] = {fc->levels * fc->features, fc->density_hidden, 1 + fc->embedding};
    if (o->dnet) mlp_init_host(dw, 3, rd, o->dnet);
    for (float* z : {o->enc_m, o->enc_v})
        if (z) std::memset(z, 0, enc * 4);
    for (float* z : {o->dnet_m, o->dnet_v})
        if (z) std::memset(z, 0, dn * 4);
    uint64_t nv = uint64_t(fc->occupancy_resolution) * fc->occupancy_resolution * fc->occupancy_resolution;
    if (o->occupancy)
        for (uint64_t i = 0; i < nv; ++i) o->occupancy[i] = 1.0f;
    o->enc_step = o->dnet_step = 0;
    return 0;
}

TFG_API int tfg_copy_bytes(tfg_ctx* c, uint64_t* h2d, uint64_t* d2h) {
    if (!c) return fail(TFG_ERR_INVALID, "copy_bytes: null context");
    if (h2d) *h2d = c->h2d_bytes;
    if (d2h) *d2h = c->d2h_bytes;
    return 0;
}

} // extern "C"

