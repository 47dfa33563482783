// TEST INFRASTRUCTURE ONLY — C-ABI glue over the reference sources compiled
// verbatim (geometry.cpp, tiler.cpp, camera.cpp, parallel.cpp, nn.hpp,
// rng.hpp from /root/reference/proj/src/core) into oracle/_ref/libtfref.so.
// Used by tests/test_oracle_vs_ref.py to pin the restatement in tf_oracle.cpp
// bit-for-bit, and by bench.py's --impl reference leg for the CPU field
// kernels.  Exceptions (tilefield::Error) become status 1.
#include "core/camera.hpp"
#include "core/geometry.hpp"
#include "core/nn.hpp"
#include "core/parallel.hpp"
#include "core/rng.hpp"
#include "core/tiler.hpp"

#include "../include/tilefield_gpu.h"

#include <cstring>
#include <vector>

using namespace tilefield;

namespace {
RationalCamera to_cam(const tfg_rpc* c) {
    RationalCamera r;
    for (int i = 0; i < 20; ++i) {
        r.line_num[i] = c->line_num[i];
        r.line_den[i] = c->line_den[i];
        r.samp_num[i] = c->samp_num[i];
        r.samp_den[i] = c->samp_den[i];
    }
    r.line_off = c->line_off;
    r.samp_off = c->samp_off;
    r.lat_off = c->lat_off;
    r.long_off = c->long_off;
    r.height_off = c->height_off;
    r.line_scale = c->line_scale;
    r.samp_scale = c->samp_scale;
    r.lat_scale = c->lat_scale;
    r.long_scale = c->long_scale;
    r.height_scale = c->height_scale;
    r.image_rows = c->image_rows;
    r.image_cols = c->image_cols;
    return r;
}
Aabb3 to_box(const double* b) { return {Vec3(b[0], b[1], b[2]), Vec3(b[3], b[4], b[5])}; }
FieldConfig to_cfg(const tfg_field_config* c) {
    FieldConfig f;
    f.levels = c->levels;
    f.table_size = c->table_size;
    f.features = c->features;
    f.n_min = c->n_min;
    f.n_max = c->n_max;
    f.density_hidden = c->density_hidden;
    f.embedding = c->embedding;
    f.color_hidden = c->color_hidden;
    f.color_layers = c->color_layers;
    f.view_freqs = c->view_freqs;
    f.density_max = c->density_max;
    f.occupancy_resolution = c->occupancy_resolution;
    f.occupancy_decay = c->occupancy_decay;
    f.occupancy_threshold = c->occupancy_threshold;
    f.occupancy_interval = c->occupancy_interval;
    return f;
}
} // namespace

extern "C" {

__attribute__((visibility("default"))) int ref_project(const tfg_rpc* c, const double* xyz,
                                                      double* rc) {
    try {
        Vec2 p = project(to_cam(c), Vec3(xyz[0], xyz[1], xyz[2]));
        rc[0] = p.x();
        rc[1] = p.y();
        return 0;
    } catch (const Error&) {
        return 1;
    }
}
__attribute__((visibility("default"))) int ref_localize(const tfg_rpc* c, const double* px,
                                                       double h, double* xy, double* resid,
                                                       int* iters) {
    try {
        LocalizeResult r = localize(to_cam(c), Vec2(px[0], px[1]), h);
        xy[0] = r.ground_xy.x();
        xy[1] = r.ground_xy.y();
        *resid = r.residual_px;
        *iters = r.iterations;
        return 0;
    } catch (const Error&) {
        return 1;
    }
}
__attribute__((visibility("default"))) int ref_ray_from_pixel(const tfg_rpc* c, int row, int col,
                                                             double zmin, double zmax, double* o,
                                                             double* d) {
    try {
        Ray r = ray_from_pixel(to_cam(c), PixelRc{row, col}, zmin, zmax, Vec3f::Zero(), 0);
        for (int k = 0; k < 3; ++k) {
            o[k] = r.origin[k];
            d[k] = r.direction[k];
        }
        return 0;
    } catch (const Error&) {
        return 1;
    }
}
__attribute__((visibility("default"))) int ref_intersect(const double* o, const double* d,
                                                        const double* box, double* t0,
                                                        double* t1) {
    Ray r;
    r.origin = Vec3(o[0], o[1], o[2]);
    r.direction = Vec3(d[0], d[1], d[2]);
    auto h = intersect_ray_aabb(r, to_box(box));
    if (!h) return 1;
    *t0 = h->first;
    *t1 = h->second;
    return 0;
}
// Segments over boxes in the given order; slot = index into boxes (TileId.col).
__attribute__((visibility("default"))) int ref_segments(const double* o, const double* d,
                                                       const double* boxes, int n, int* slot,
                                                       double* tn, double* tf) {
    try {
        std::vector<TileBox> tb;
        for (int i = 0; i < n; ++i) tb.push_back({TileId{0, i}, to_box(boxes + 6 * i)});
        TileBoxSet set(tb);
        Ray r;
        r.origin = Vec3(o[0], o[1], o[2]);
        r.direction = Vec3(d[0], d[1], d[2]);
        auto segs = set.segments(r);
        for (size_t k = 0; k < segs.size(); ++k) {
            slot[k] = segs[k].tile_id.col;
            tn[k] = segs[k].t_near;
            tf[k] = segs[k].t_far;
        }
        return int(segs.size());
    } catch (const Error&) {
        return -1;
    }
}
__attribute__((visibility("default"))) int ref_grid_edges(const tfg_roi* roi, int rows, int cols,
                                                         double* east, double* north) {
    try {
        Roi r{roi->easting_min, roi->easting_max, roi->northing_min,
              roi->northing_max, roi->z_min,      roi->z_max};
        TileGrid g = TileGrid::build(r, rows, cols);
        for (int k = 0; k <= cols; ++k) east[k] = g.boundary_easting(k);
        for (int k = 0; k <= rows; ++k) north[k] = g.boundary_northing(k);
        return 0;
    } catch (const Error&) {
        return 1;
    }
}
__attribute__((visibility("default"))) int ref_tile_frame(const tfg_roi* roi, int rows, int cols,
                                                         int r, int c, double* box6,
                                                         double* inv3) {
    Roi rr{roi->easting_min, roi->easting_max, roi->northing_min,
           roi->northing_max, roi->z_min,      roi->z_max};
    TileGrid g = TileGrid::build(rr, rows, cols);
    const Tile& t = g.tile(r, c);
    for (int k = 0; k < 3; ++k) {
        box6[k] = t.box.min_corner[k];
        box6[3 + k] = t.box.max_corner[k];
        inv3[k] = t.local_frame.inv_size[k];
    }
    return 0;
}
__attribute__((visibility("default"))) int ref_to_local(const tfg_roi* roi, int rows, int cols,
                                                       int r, int c, const double* p,
                                                       double* out) {
    Roi rr{roi->easting_min, roi->easting_max, roi->northing_min,
           roi->northing_max, roi->z_min,      roi->z_max};
    TileGrid g = TileGrid::build(rr, rows, cols);
    Vec3 q = g.tile(r, c).local_frame.to_local(Vec3(p[0], p[1], p[2]));
    for (int k = 0; k < 3; ++k) out[k] = q[k];
    return 0;
}
__attribute__((visibility("default"))) int ref_candidate_tiles(const tfg_roi* roi, int rows,
                                                              int cols, const double* o,
                                                              const double* d, int* pairs,
                                                              int capacity) {
    Roi rr{roi->easting_min, roi->easting_max, roi->northing_min,
           roi->northing_max, roi->z_min,      roi->z_max};
    TileGrid g = TileGrid::build(rr, rows, cols);
    Ray r;
    r.origin = Vec3(o[0], o[1], o[2]);
    r.direction = Vec3(d[0], d[1], d[2]);
    auto ids = g.candidate_tiles(r);
    for (size_t k = 0; k < ids.size() && int(k) < capacity; ++k) {
        pairs[2 * k] = ids[k].row;
        pairs[2 * k + 1] = ids[k].col;
    }
    return int(ids.size());
}
__attribute__((visibility("default"))) int ref_crop_for_tile(const tfg_rpc* c, const double* box,
                                                            int margin, int* rect) {
    try {
        auto cr = crop_for_tile(to_cam(c), to_box(box), margin, 0, TileId{0, 0});
        if (!cr) return 1;
        rect[0] = cr->row_min;
        rect[1] = cr->row_max;
        rect[2] = cr->col_min;
        rect[3] = cr->col_max;
        return 0;
    } catch (const Error&) {
        return 2;
    }
}
__attribute__((visibility("default"))) int ref_level_resolution(const tfg_field_config* c,
                                                               int level) {
    return level_resolution(to_cfg(c), level);
}
__attribute__((visibility("default"))) uint64_t ref_splitmix64(uint64_t x) {
    return splitmix64(x);
}
__attribute__((visibility("default"))) uint64_t ref_hash_combine(uint64_t a, uint64_t b) {
    return hash_combine(a, b);
}
// n draws of Rng(seed): kind 0 u64, 1 double, 2 float (as double), 3 below(arg)
__attribute__((visibility("default"))) void ref_rng_draws(uint64_t seed, int kind, uint64_t arg,
                                                         int n, uint64_t* u, double* f) {
    Rng r(seed);
    for (int i = 0; i < n; ++i) {
        switch (kind) {
        case 0: u[i] = r.next_u64(); break;
        case 1: f[i] = r.next_double(); break;
        case 2: f[i] = r.next_float(); break;
        default: u[i] = r.next_below(arg); break;
        }
    }
}
// MlpT<float>::init with Rng(seed); writes params.
__attribute__((visibility("default"))) int ref_mlp_init(const int* widths, int nw, uint64_t seed,
                                                       float* params) {
    MlpT<float> m;
    Rng r(seed);
    m.init(std::vector<int>(widths, widths + nw), r);
    std::memcpy(params, m.params.data(), m.params.size() * 4);
    return int(m.params.size());
}
// MlpT<float>::forward_p / backward_p for one input; grad accumulates.
__attribute__((visibility("default"))) int ref_mlp_fwd_bwd(const int* widths, int nw,
                                                          const float* params, const float* x,
                                                          float* out, const float* d_out,
                                                          float* grad, float* d_in) {
    MlpT<float> m;
    m.widths.assign(widths, widths + nw);
    std::vector<float> acts(MlpT<float>::act_count(m.widths));
    const float* o = m.forward_p(params, x, acts.data());
    for (int i = 0; i < m.out_dim(); ++i) out[i] = o[i];
    if (d_out) {
        int maxw = 0;
        for (int w : m.widths) maxw = std::max(maxw, w);
        std::vector<float> scratch(2 * maxw);
        m.backward_p(params, acts.data(), d_out, grad, d_in, scratch.data());
    }
    return 0;
}
// HashGridT<float>::init with Rng(seed) -> tables; lookup / backward.
__attribute__((visibility("default"))) uint64_t ref_hash_init(const tfg_field_config* c,
                                                             uint64_t seed, float* tables) {
    HashGridT<float> g;
    Rng r(seed);
    g.init(to_cfg(c), r);
    if (tables) std::memcpy(tables, g.tables.data(), g.tables.size() * 4);
    return g.tables.size();
}
__attribute__((visibility("default"))) int ref_hash_lookup_bwd(const tfg_field_config* c,
                                                              const float* tables, int n_points,
                                                              const float* p3, float* out,
                                                              const float* d_out, float* grad) {
    HashGridT<float> g;
    Rng r(0);
    g.init(to_cfg(c), r);
    for (int i = 0; i < n_points; ++i) {
        g.lookup_p(tables, p3 + 3 * i, out + size_t(i) * c->levels * c->features);
        if (d_out && grad) g.backward(p3 + 3 * i, d_out + size_t(i) * c->levels * c->features, grad);
    }
    return 0;
}
__attribute__((visibility("default"))) float ref_density_activation(float raw, float maxd,
                                                                   float* draw) {
    return density_activation<float>(raw, maxd, draw);
}
__attribute__((visibility("default"))) void ref_encode_direction(const float* d, int freqs,
                                                                float* out) {
    encode_direction<float>(d, freqs, out);
}
__attribute__((visibility("default"))) void ref_chunk_range(uint64_t n, int workers, int c,
                                                           uint64_t* b, uint64_t* e) {
    auto r = chunk_range(n, workers, c);
    *b = r.first;
    *e = r.second;
}

} // extern "C"
