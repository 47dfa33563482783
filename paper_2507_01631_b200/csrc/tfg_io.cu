// tfg_io.cu — persistence behind the C-ABI: tile / colour checkpoints and
// run save/resume (field.hpp:202-210) and the crop cache
// (build_crop_cache).  Host file I/O over the context's
// pinned host records and images.
#include "tfg_internal.h"

// ---------------------------------------------------------------- checkpoints
namespace {
constexpr char kCkptMagic[8] = {'T', 'F', 'C', 'K', 'P', 'T', '0', '1'};
constexpr uint32_t kCkptVersion = 1;

bool same_cfg(const tfg_field_config& a, const tfg_field_config& b) {
    return std::memcmp(&a, &b, sizeof(a)) == 0;
}

int write_ckpt(const char* path, uint32_t kind, const tfg_field_config& cfg, int row, int col,
               uint64_t n_params, uint64_t n_occ, uint64_t step0, uint64_t step1,
               const float* const* arrays, const uint64_t* counts, int n_arrays) {
    std::ofstream f(path, std::ios::binary);
    if (!f) return fail(TFG_ERR_INVALID, std::string("checkpoint: cannot open ") + path);
    int32_t rc2[2] = {row, col};
    uint64_t hdr[4] = {n_params, n_occ, step0, step1};
    f.write(kCkptMagic, 8);
    f.write(reinterpret_cast<const char*>(&kCkptVersion), 4);
    f.write(reinterpret_cast<const char*>(&kind), 4);
    f.write(reinterpret_cast<const char*>(&cfg), sizeof(cfg));
    f.write(reinterpret_cast<const char*>(rc2), 8);
    f.write(reinterpret_cast<const char*>(hdr), 32);
    for (int i = 0; i < n_arrays; ++i) {
        static const std::vector<float> zeros(1 << 16, 0.f);
        if (arrays[i]) {
            f.write(reinterpret_cast<const char*>(arrays[i]), counts[i] * 4);
        } else {  // absent moments are written as zeros
            for (uint64_t k = 0; k < counts[i]; k += zeros.size())
                f.write(reinterpret_cast<const char*>(zeros.data()),
                        std::min<uint64_t>(zeros.size(), counts[i] - k) * 4);
        }
    }
    if (!f.good()) return fail(TFG_ERR_INVALID, std::string("checkpoint: write failed for ") + path);
    return 0;
}

int read_ckpt_header(std::ifstream& f, const char* path, uint32_t kind, const tfg_field_config& cfg,
                     int* row, int* col, uint64_t* hdr) {
    char magic[8];
    uint32_t ver = 0, k = 0;
    tfg_field_config c{};
    int32_t rc2[2];
    f.read(magic, 8);
    f.read(reinterpret_cast<char*>(&ver), 4);
    f.read(reinterpret_cast<char*>(&k), 4);
    f.read(reinterpret_cast<char*>(&c), sizeof(c));
    f.read(reinterpret_cast<char*>(rc2), 8);
    f.read(reinterpret_cast<char*>(hdr), 32);
    if (!f.good() || std::memcmp(magic, kCkptMagic, 8) != 0)
        return fail(TFG_ERR_INVALID, std::string("checkpoint: bad magic in ") + path);
    if (ver != kCkptVersion || k != kind)
        return fail(TFG_ERR_INVALID, std::string("checkpoint: unsupported version/kind in ") + path);
    if (!same_cfg(c, cfg))
        return fail(TFG_ERR_INVALID, std::string("checkpoint: FieldConfig mismatch in ") + path);
    if (row) *row = rc2[0];
    if (col) *col = rc2[1];
    return 0;
}

// The payload must be exactly the arrays the header announces: checked
// against the file size before anything is read into caller buffers.
int read_arrays(std::ifstream& f, const char* path, float* const* arrays, const uint64_t* counts, int n) {
    const std::streamoff here = f.tellg();
    f.seekg(0, std::ios::end);
    const std::streamoff end = f.tellg();
    f.seekg(here, std::ios::beg);
    uint64_t need = 0;
    for (int i = 0; i < n; ++i) need += counts[i] * 4;
    if (here < 0 || end < here || uint64_t(end - here) != need)
        return fail(TFG_ERR_INVALID, std::string("checkpoint: payload size does not match the header in ") + path);
    for (int i = 0; i < n; ++i) {
        if (arrays[i]) {
            f.read(reinterpret_cast<char*>(arrays[i]), counts[i] * 4);
        } else {
            f.seekg(std::streamoff(counts[i] * 4), std::ios::cur);
        }
    }
    if (!f.good()) return fail(TFG_ERR_INVALID, std::string("checkpoint: truncated ") + path);
    return 0;
}
} // namespace

extern "C" {

TFG_API int tfg_save_tile_checkpoint(const char* path, const tfg_field_config* cfg, int row, int col,
                                     const tfg_tile_state* st) {
    uint64_t enc, dn;
    tfg_param_counts(cfg, &enc, &dn, nullptr);
    uint64_t occ = uint64_t(cfg->occupancy_resolution) * cfg->occupancy_resolution * cfg->occupancy_resolution;
    const float* arr[7] = {st->enc, st->dnet, st->enc_m, st->enc_v, st->dnet_m, st->dnet_v, st->occupancy};
    const uint64_t cnt[7] = {enc, dn, enc, enc, dn, dn, occ};
    if (!st->enc || !st->dnet || !st->occupancy)
        return fail(TFG_ERR_INVALID, "save_tile_checkpoint: params and occupancy are required");
    return write_ckpt(path, 1, *cfg, row, col, enc + dn, occ, st->enc_step, st->dnet_step, arr, cnt, 7);
}

TFG_API int tfg_load_tile_checkpoint(const char* path, const tfg_field_config* cfg, int* row, int* col,
                                     tfg_tile_state* st) {
    std::ifstream f(path, std::ios::binary);
    if (!f) return fail(TFG_ERR_INVALID, std::string("checkpoint: cannot open ") + path);
    uint64_t hdr[4];
    int rc = read_ckpt_header(f, path, 1, *cfg, row, col, hdr);
    if (rc) return rc;
    uint64_t enc, dn;
    tfg_param_counts(cfg, &enc, &dn, nullptr);
    if (hdr[0] != enc + dn) return fail(TFG_ERR_INVALID, "checkpoint: parameter count mismatch");
    // the occupancy count is stored apart from the FieldConfig: it must be
    // exactly res^3 (the caller's buffer size)
    const uint64_t occ =
        uint64_t(cfg->occupancy_resolution) * cfg->occupancy_resolution * cfg->occupancy_resolution;
    if (hdr[1] != occ) return fail(TFG_ERR_INVALID, "checkpoint: occupancy count mismatch");
    float* arr[7] = {st->enc, st->dnet, st->enc_m, st->enc_v, st->dnet_m, st->dnet_v, st->occupancy};
    const uint64_t cnt[7] = {enc, dn, enc, enc, dn, dn, occ};
    rc = read_arrays(f, path, arr, cnt, 7);
    if (rc) return rc;
    st->enc_step = hdr[2];
    st->dnet_step = hdr[3];
    return 0;
}

TFG_API int tfg_save_color_checkpoint(const char* path, const tfg_field_config* cfg, const float* params,
                                      const float* m, const float* v, uint64_t step) {
    uint64_t col;
    tfg_param_counts(cfg, nullptr, nullptr, &col);
    const float* arr[3] = {params, m, v};
    const uint64_t cnt[3] = {col, col, col};
    return write_ckpt(path, 2, *cfg, -1, -1, col, 0, step, 0, arr, cnt, 3);
}

TFG_API int tfg_load_color_checkpoint(const char* path, const tfg_field_config* cfg, float* params,
                                      float* m, float* v, uint64_t* step) {
    std::ifstream f(path, std::ios::binary);
    if (!f) return fail(TFG_ERR_INVALID, std::string("checkpoint: cannot open ") + path);
    uint64_t hdr[4];
    int rc = read_ckpt_header(f, path, 2, *cfg, nullptr, nullptr, hdr);
    if (rc) return rc;
    uint64_t col;
    tfg_param_counts(cfg, nullptr, nullptr, &col);
    if (hdr[0] != col || hdr[1] != 0) return fail(TFG_ERR_INVALID, "checkpoint: parameter count mismatch");
    float* arr[3] = {params, m, v};
    const uint64_t cnt[3] = {col, col, col};
    rc = read_arrays(f, path, arr, cnt, 3);
    if (rc) return rc;
    if (step) *step = hdr[2];
    return 0;
}

// Saves the run: the window slots are copied back to their host records
// first, then every record that was ever materialised and the colour net.
TFG_API int tfg_save_run(tfg_ctx* c, const char* dir) {
    if (!c || c->n_views == 0) return fail(TFG_ERR_STATE, "save_run: no scene");
    CK(cudaSetDevice(c->device));
    if (settle_steps(c)) return TFG_ERR_CUDA;  // saved step counts exclude skipped steps
    CK(cudaEventRecord(c->ev_main, c->st));
    CK(cudaStreamWaitEvent(c->side, c->ev_main, 0));
    for (int s = 0; s < c->nslots; ++s)
        if (slot_copy(c, s, c->slot_tile[s], true)) return TFG_ERR_CUDA;
    CK(cudaStreamSynchronize(c->side));
    std::string d(dir);
    for (size_t ti = 0; ti < c->tiles.size(); ++ti) {
        TileHost& t = c->tiles[ti];
        if (!c->init.ready[ti].load() || !t.created) continue;
        float* p = t.rec;
        tfg_tile_state st{};
        st.enc = p;
        st.dnet = p + c->dn_off;
        st.enc_m = p + c->stride;
        st.dnet_m = p + c->stride + c->dn_off;
        st.enc_v = p + 2 * c->stride;
        st.dnet_v = p + 2 * c->stride + c->dn_off;
        st.occupancy = p + 3 * c->stride;
        st.enc_step = t.enc_step;
        st.dnet_step = t.dnet_step;
        char name[64];
        std::snprintf(name, sizeof name, "/tiles/r%d_c%d.ckpt", int(ti) / c->cols, int(ti) % c->cols);
        int rc = tfg_save_tile_checkpoint((d + name).c_str(), &c->fc, int(ti) / c->cols,
                                          int(ti) % c->cols, &st);
        if (rc) return rc;
    }
    uint64_t n = c->n_params - c->color_off;
    std::vector<float> p(n), m(n), v(n);
    int rc = tfg_get_color(c, p.data(), m.data(), v.data(), nullptr);
    if (rc) return rc;
    return tfg_save_color_checkpoint((d + "/color_net.ckpt").c_str(), &c->fc, p.data(), m.data(), v.data(),
                                     c->color_step);
}

// Restores a saved run into the host records (tiles absent from `dir` keep
// their fresh initialisation) and the colour net; call before set_window.
TFG_API int tfg_load_run(tfg_ctx* c, const char* dir) {
    if (!c || c->n_views == 0) return fail(TFG_ERR_STATE, "load_run: no scene");
    if (c->nslots) return fail(TFG_ERR_STATE, "load_run: call before the first set_window");
    std::string d(dir);
    for (size_t ti = 0; ti < c->tiles.size(); ++ti) {
        char name[64];
        std::snprintf(name, sizeof name, "/tiles/r%d_c%d.ckpt", int(ti) / c->cols, int(ti) % c->cols);
        std::string path = d + name;
        std::ifstream probe(path, std::ios::binary);
        if (!probe) continue;
        probe.close();
        if (ensure_record(c, int(ti))) return TFG_ERR_CUDA;
        TileHost& t = c->tiles[ti];
        float* p = t.rec;
        tfg_tile_state st{};
        st.enc = p;
        st.dnet = p + c->dn_off;
        st.enc_m = p + c->stride;
        st.dnet_m = p + c->stride + c->dn_off;
        st.enc_v = p + 2 * c->stride;
        st.dnet_v = p + 2 * c->stride + c->dn_off;
        st.occupancy = p + 3 * c->stride;
        int row, col;
        int rc = tfg_load_tile_checkpoint(path.c_str(), &c->fc, &row, &col, &st);
        if (rc) return rc;
        if (row * c->cols + col != int(ti)) return fail(TFG_ERR_INVALID, "load_run: tile id mismatch in " + path);
        t.enc_step = st.enc_step;
        t.dnet_step = st.dnet_step;
    }
    uint64_t n = c->n_params - c->color_off;
    std::vector<float> p(n), m(n), v(n);
    uint64_t step = 0;
    int rc = tfg_load_color_checkpoint((d + "/color_net.ckpt").c_str(), &c->fc, p.data(), m.data(), v.data(),
                                       &step);
    if (rc) return rc;
    return tfg_set_color(c, p.data(), m.data(), v.data(), step);
}

} // extern "C"

// ---------------------------------------------------------------- crop cache
namespace {
constexpr char kCropMagic[8] = {'T', 'F', 'C', 'R', 'O', 'P', '0', '1'};
struct CropEntry {
    int32_t view, row, col, r0, r1, c0, c1, pad;
    uint64_t offset, bytes;
};
static_assert(sizeof(CropEntry) == 48, "crop index entry");

void crop_index(const tfg_ctx* c, std::vector<CropEntry>& idx) {
    idx.clear();
    uint64_t off = 0;
    for (int v = 0; v < c->n_views; ++v)
        for (int ti = 0; ti < c->rows * c->cols; ++ti) {
            CropEntry e{};
            e.view = v;
            e.row = ti / c->cols;
            e.col = ti % c->cols;
            double b[6];
            tile_box(c, ti, b);
            Crop cr;
            if (crop_for_tile(c->cams[v], b, c->tc.margin_px, &cr)) {
                e.r0 = cr.r0;
                e.r1 = cr.r1;
                e.c0 = cr.c0;
                e.c1 = cr.c1;
                e.offset = off;
                e.bytes = uint64_t(cr.r1 - cr.r0) * uint64_t(cr.c1 - cr.c0) * 3;
                off += e.bytes;
            }
            idx.push_back(e);
        }
}
} // namespace

extern "C" {

TFG_API int tfg_crop_rect(tfg_ctx* c, int view, int row, int col, int32_t* out) {
    if (!c || c->n_views == 0) return fail(TFG_ERR_STATE, "crop_rect: call set_scene first");
    if (view < 0 || view >= c->n_views || row < 0 || row >= c->rows || col < 0 || col >= c->cols || !out)
        return fail(TFG_ERR_INVALID, "crop_rect: bad view or tile");
    double b[6];
    tile_box(c, row * c->cols + col, b);
    Crop cr;
    if (!crop_for_tile(c->cams[view], b, c->tc.margin_px, &cr)) cr = Crop{};
    out[0] = cr.r0;
    out[1] = cr.r1;
    out[2] = cr.c0;
    out[3] = cr.c1;
    return 0;
}

TFG_API int tfg_build_crop_cache(tfg_ctx* c, const char* path, uint64_t* total) {
    if (!c || c->n_views == 0) return fail(TFG_ERR_STATE, "build_crop_cache: call set_scene first");
    std::vector<CropEntry> idx;
    crop_index(c, idx);
    std::ofstream f(path, std::ios::binary);
    if (!f) return fail(TFG_ERR_INVALID, std::string("crop cache: cannot open ") + path);
    uint32_t hdr32[6] = {1u, uint32_t(c->n_views), uint32_t(c->rows), uint32_t(c->cols),
                         uint32_t(c->tc.margin_px), 0u};
    uint64_t n = idx.size(), data_off = 8 + sizeof(hdr32) + 16 + n * sizeof(CropEntry);
    f.write(kCropMagic, 8);
    f.write(reinterpret_cast<const char*>(hdr32), sizeof(hdr32));
    f.write(reinterpret_cast<const char*>(&n), 8);
    f.write(reinterpret_cast<const char*>(&data_off), 8);
    f.write(reinterpret_cast<const char*>(idx.data()), n * sizeof(CropEntry));
    uint64_t tot = 0;
    for (const CropEntry& e : idx) {
        if (!e.bytes) continue;
        const uint8_t* im = c->h_images[e.view];
        size_t W = size_t(c->cams[e.view].image_cols);
        for (int r = e.r0; r < e.r1; ++r)
            f.write(reinterpret_cast<const char*>(im + 3 * (size_t(r) * W + size_t(e.c0))),
                    std::streamsize(3 * (e.c1 - e.c0)));
        tot += e.bytes;
    }
    if (!f.good()) return fail(TFG_ERR_INVALID, std::string("crop cache: write failed for ") + path);
    if (total) *total = tot;
    return 0;
}

TFG_API int tfg_load_crop_cache(tfg_ctx* c, const char* path) {
    if (!c || c->n_views == 0) return fail(TFG_ERR_STATE, "load_crop_cache: call set_scene first");
    if (c->nslots) return fail(TFG_ERR_STATE, "load_crop_cache: call before the first set_window");
    std::ifstream f(path, std::ios::binary);
    if (!f) return fail(TFG_ERR_INVALID, std::string("crop cache: cannot open ") + path);
    char magic[8];
    uint32_t hdr32[6];
    uint64_t n = 0, data_off = 0;
    f.read(magic, 8);
    f.read(reinterpret_cast<char*>(hdr32), sizeof(hdr32));
    f.read(reinterpret_cast<char*>(&n), 8);
    f.read(reinterpret_cast<char*>(&data_off), 8);
    if (!f.good() || std::memcmp(magic, kCropMagic, 8) != 0 || hdr32[0] != 1u)
        return fail(TFG_ERR_INVALID, std::string("crop cache: bad header in ") + path);
    if (hdr32[1] != uint32_t(c->n_views) || hdr32[2] != uint32_t(c->rows) || hdr32[3] != uint32_t(c->cols) ||
        hdr32[4] != uint32_t(c->tc.margin_px))
        return fail(TFG_ERR_INVALID, "crop cache: views / grid / margin differ from the scene");
    std::vector<CropEntry> want, got(n);
    crop_index(c, want);
    f.read(reinterpret_cast<char*>(got.data()), std::streamsize(n * sizeof(CropEntry)));
    if (!f.good() || n != want.size() ||
        std::memcmp(got.data(), want.data(), n * sizeof(CropEntry)) != 0)
        return fail(TFG_ERR_INVALID, "crop cache: index differs from this scene's crop_for_tile rects");
    std::vector<uint8_t> buf;
    for (const CropEntry& e : got) {
        if (!e.bytes) continue;
        buf.resize(e.bytes);
        f.seekg(std::streamoff(data_off + e.offset));
        f.read(reinterpret_cast<char*>(buf.data()), std::streamsize(e.bytes));
        if (!f.good()) return fail(TFG_ERR_INVALID, std::string("crop cache: truncated ") + path);
        uint8_t* im = c->h_images[e.view];
        size_t W = size_t(c->cams[e.view].image_cols), w3 = size_t(3 * (e.c1 - e.c0));
        for (int r = e.r0; r < e.r1; ++r)
            std::memcpy(im + 3 * (size_t(r) * W + size_t(e.c0)), buf.data() + size_t(r - e.r0) * w3, w3);
    }
    return 0;
}

} // extern "C"
