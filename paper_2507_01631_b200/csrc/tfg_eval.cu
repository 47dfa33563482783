// tfg_eval.cu — evaluation behind the C-ABI (evalio):
// PSNR / SSIM / depth MAE / tile-edge band mask on the GPU (k_eval.cu) and the
// full-frame render (cmd_render).
#include "tfg_internal.h"

// ---------------------------------------------------------------- evaluation
namespace {
// Stream-ordered device scratch of one call, released on every exit path.
struct Scratch {
    tfg_ctx* c;
    std::vector<void*> ptrs;
    explicit Scratch(tfg_ctx* ctx) : c(ctx) {}
    ~Scratch() {
        for (void* p : ptrs) cudaFreeAsync(p, c->st);
    }
    template <typename T>
    int alloc(T** d, uint64_t n) {
        CK(cudaMallocAsync(reinterpret_cast<void**>(d), n * sizeof(T), c->st));
        ptrs.push_back(*d);
        return 0;
    }
    template <typename T>
    int upload(T** d, const T* h, uint64_t n) {
        if (alloc(d, n)) return TFG_ERR_CUDA;
        CK(cudaMemcpyAsync(*d, h, n * sizeof(T), cudaMemcpyHostToDevice, c->st));
        return 0;
    }
};
} // namespace

extern "C" {

TFG_API int tfg_psnr(tfg_ctx* c, const float* a, const float* b, uint64_t n, double* db) {
    if (!c || !a || !b || n == 0 || !db) return fail(TFG_ERR_INVALID, "psnr: empty or null input");
    CK(cudaSetDevice(c->device));
    Scratch sc(c);
    float *da = nullptr, *dbuf = nullptr;
    double* acc = nullptr;
    if (sc.upload(&da, a, n) || sc.upload(&dbuf, b, n) || sc.alloc(&acc, 1)) return TFG_ERR_CUDA;
    CK(cudaMemsetAsync(acc, 0, 8, c->st));
    launch_sq_diff(da, dbuf, n, acc, c->sms, c->st);
    c->launches += 1;
    double s = 0.0;
    CK(cudaMemcpyAsync(&s, acc, 8, cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
    double mse = s / double(n);
    *db = mse > 0.0 ? std::min(99.0, 10.0 * std::log10(1.0 / mse)) : 99.0;
    return 0;
}

TFG_API int tfg_ssim(tfg_ctx* c, const float* a, const float* b, int rows, int cols, double* out) {
    if (!c || !a || !b || !out) return fail(TFG_ERR_INVALID, "ssim: null input");
    if (rows < 11 || cols < 11) return fail(TFG_ERR_INVALID, "ssim: image smaller than the 11x11 window");
    CK(cudaSetDevice(c->device));
    uint64_t n = uint64_t(rows) * uint64_t(cols) * 3;
    Scratch sc(c);
    float *da = nullptr, *dbuf = nullptr, *gw = nullptr;
    double* acc = nullptr;
    if (sc.upload(&da, a, n) || sc.upload(&dbuf, b, n)) return TFG_ERR_CUDA;
    float w[11];
    {
        double g[11], sum = 0.0;
        for (int k = 0; k < 11; ++k) {
            double x = k - 5;
            g[k] = std::exp(-(x * x) / (2.0 * 1.5 * 1.5));
            sum += g[k];
        }
        for (int k = 0; k < 11; ++k) w[k] = float(g[k] / sum);
    }
    if (sc.upload(&gw, static_cast<const float*>(w), 11) || sc.alloc(&acc, 1)) return TFG_ERR_CUDA;
    CK(cudaMemsetAsync(acc, 0, 8, c->st));
    launch_ssim(da, dbuf, rows, cols, gw, acc, c->st);
    c->launches += 1;
    double s = 0.0;
    CK(cudaMemcpyAsync(&s, acc, 8, cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
    *out = s / (double(rows - 10) * double(cols - 10));
    return 0;
}

TFG_API int tfg_depth_mae(tfg_ctx* c, const float* d1, const float* d2, const uint8_t* mask, uint64_t n,
                          double* out) {
    if (!c || !d1 || !d2 || n == 0 || !out) return fail(TFG_ERR_INVALID, "depth_mae: empty or null input");
    CK(cudaSetDevice(c->device));
    Scratch sc(c);
    float *a = nullptr, *b = nullptr;
    uint8_t* m = nullptr;
    double* acc = nullptr;
    if (sc.upload(&a, d1, n) || sc.upload(&b, d2, n) || sc.alloc(&acc, 2)) return TFG_ERR_CUDA;
    if (mask && sc.upload(&m, mask, n)) return TFG_ERR_CUDA;
    CK(cudaMemsetAsync(acc, 0, 16, c->st));
    launch_abs_diff(a, b, m, n, acc, c->sms, c->st);
    c->launches += 1;
    double s[2] = {0.0, 0.0};
    CK(cudaMemcpyAsync(s, acc, 16, cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
    if (s[1] == 0.0) return fail(TFG_ERR_INVALID, "depth_mae: empty mask");
    *out = s[0] / s[1];
    return 0;
}

TFG_API int tfg_edge_band_mask(tfg_ctx* c, const tfg_rpc* cam, int band_px, uint8_t* mask) {
    if (!c || c->n_views == 0) return fail(TFG_ERR_STATE, "edge_band_mask: call set_scene first");
    if (!cam || !mask || band_px < 0) return fail(TFG_ERR_INVALID, "edge_band_mask: bad arguments");
    CK(cudaSetDevice(c->device));
    uint64_t npx = uint64_t(cam->image_rows) * uint64_t(cam->image_cols);
    Scratch sc(c);
    uint8_t* dm = nullptr;
    tfg_rpc* dcam = nullptr;
    if (sc.alloc(&dm, npx) || sc.upload(&dcam, cam, 1)) return TFG_ERR_CUDA;
    CK(cudaMemsetAsync(dm, 0, npx, c->st));
    // sample the boundary lines at 1/8 of the view's ground footprint per pixel
    double ext = std::max(c->roi.easting_max - c->roi.easting_min, c->roi.northing_max - c->roi.northing_min);
    double gsd = std::fabs(cam->long_scale) / std::max(1.0, std::fabs(cam->samp_scale));
    double step = std::max(gsd / 8.0, ext / 1.0e6);
    uint64_t per_line = uint64_t(ext / step) + 2;
    launch_edge_band(dcam, c->d_east, c->d_north, c->rows, c->cols, c->roi.z_min, c->roi.z_max, step, per_line,
                     band_px, dm, c->st);
    c->launches += 1;
    CK(cudaMemcpyAsync(mask, dm, npx, cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
    return 0;
}

TFG_API int tfg_render_view(tfg_ctx* c, const tfg_rpc* cam, float* rgb, float* depth, float* opacity) {
    if (!c || !cam) return fail(TFG_ERR_INVALID, "render_view: null input");
    uint64_t npx = uint64_t(cam->image_rows) * uint64_t(cam->image_cols);
    const uint64_t chunk = 1u << 22;
    std::vector<int32_t> px;
    for (uint64_t p0 = 0; p0 < npx; p0 += chunk) {
        uint64_t nb = std::min<uint64_t>(chunk, npx - p0);
        px.resize(2 * nb);
        for (uint64_t i = 0; i < nb; ++i) {
            px[2 * i] = int32_t((p0 + i) / uint64_t(cam->image_cols));
            px[2 * i + 1] = int32_t((p0 + i) % uint64_t(cam->image_cols));
        }
        int rc = tfg_render_pixels(c, cam, px.data(), int(nb), rgb ? rgb + 3 * p0 : nullptr,
                                   depth ? depth + p0 : nullptr, opacity ? opacity + p0 : nullptr);
        if (rc) return rc;
    }
    return 0;
}

} // extern "C"
