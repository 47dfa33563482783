// k_eval.cu — evaluation metrics of the render path (§8(f) row 2; evalio
// module): PSNR, SSIM, depth MAE and the tile-edge band mask
// of the boundary-band depth MAE.  All are HBM-bound reductions; sums are
// accumulated in FP64.
//
//   psnr  = min(99, 10 log10(1 / MSE)) over all channels, 99 dB if MSE == 0
//   ssim  = mean over the 'valid' windows of the local SSIM of the channel-mean
//           grey images, 11x11 Gaussian (sigma 1.5, normalised), K1 0.01,
//           K2 0.03, L 1
//   mae   = mean |d1 - d2| over the mask
//   band  = pixels within +-B px (Chebyshev) of the projected tile edges
//           (the grid's boundary lines at z_min and at z_max, sampled every
//           1/8 of the view's pixel footprint; pinned in DESIGN.md)
#include <cuda_runtime.h>

#include "tf_common.cuh"
#include "tf_kernels.h"

namespace tfg {

namespace {

__device__ __forceinline__ double block_sum(double v) {
    __shared__ double part[32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int nw = (blockDim.x * blockDim.y + 31) >> 5;
    const int tid = threadIdx.y * blockDim.x + threadIdx.x;
    const int w = tid >> 5, l = tid & 31;
    if (l == 0) part[w] = v;
    __syncthreads();
    double s = 0.0;
    if (tid < 32) {
        s = tid < nw ? part[tid] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    }
    return s;  // valid in thread 0
}

__global__ void sq_diff_kernel(const float* __restrict__ a, const float* __restrict__ b, uint64_t n,
                               double* __restrict__ out) {
    double s = 0.0;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x) {
        double d = double(a[i]) - double(b[i]);
        s += d * d;
    }
    s = block_sum(s);
    if (threadIdx.x == 0) atomicAdd(out, s);
}

__global__ void abs_diff_kernel(const float* __restrict__ a, const float* __restrict__ b,
                                const uint8_t* __restrict__ mask, uint64_t n, double* __restrict__ out) {
    double s = 0.0, c = 0.0;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x) {
        if (mask && !mask[i]) continue;
        s += fabs(double(a[i]) - double(b[i]));
        c += 1.0;
    }
    s = block_sum(s);
    __syncthreads();
    c = block_sum(c);
    if (threadIdx.x == 0) {
        atomicAdd(out, s);
        atomicAdd(out + 1, c);
    }
}

constexpr int kWin = 11, kHalo = kWin - 1, kTile = 32;

// One block per 32x32 tile of SSIM windows (window top-left corners); the
// (32+10)^2 grey patches of both images are staged in smem, blurred
// horizontally then vertically.
__global__ void __launch_bounds__(256) ssim_kernel(const float* __restrict__ a, const float* __restrict__ b,
                                                   int rows, int cols, const float* __restrict__ gw,
                                                   double* __restrict__ out) {
    __shared__ float ga[kTile + kHalo][kTile + kHalo], gb[kTile + kHalo][kTile + kHalo];
    __shared__ float h[5][kTile + kHalo][kTile];
    const int R = rows - kHalo, C = cols - kHalo;  // number of valid windows per axis
    const int r0 = blockIdx.y * kTile, c0 = blockIdx.x * kTile;
    const int tid = threadIdx.y * blockDim.x + threadIdx.x, nth = blockDim.x * blockDim.y;
    for (int i = tid; i < (kTile + kHalo) * (kTile + kHalo); i += nth) {
        int y = i / (kTile + kHalo), x = i % (kTile + kHalo);
        int gy = r0 + y, gx = c0 + x;
        float va = 0.f, vb = 0.f;
        if (gy < rows && gx < cols) {
            const float* pa = a + 3 * (uint64_t(gy) * cols + gx);
            const float* pb = b + 3 * (uint64_t(gy) * cols + gx);
            va = (pa[0] + pa[1] + pa[2]) / 3.f;  // grey = channel mean
            vb = (pb[0] + pb[1] + pb[2]) / 3.f;
        }
        ga[y][x] = va;
        gb[y][x] = vb;
    }
    __syncthreads();
    for (int i = tid; i < (kTile + kHalo) * kTile; i += nth) {
        int y = i / kTile, x = i % kTile;
        float m0 = 0.f, m1 = 0.f, m2 = 0.f, m3 = 0.f, m4 = 0.f;
#pragma unroll
        for (int k = 0; k < kWin; ++k) {
            float w = gw[k], p = ga[y][x + k], q = gb[y][x + k];
            m0 += w * p;
            m1 += w * q;
            m2 += w * p * p;
            m3 += w * q * q;
            m4 += w * p * q;
        }
        h[0][y][x] = m0;
        h[1][y][x] = m1;
        h[2][y][x] = m2;
        h[3][y][x] = m3;
        h[4][y][x] = m4;
    }
    __syncthreads();
    const float C1 = 0.01f * 0.01f, C2 = 0.03f * 0.03f;
    double s = 0.0;
    for (int i = tid; i < kTile * kTile; i += nth) {
        int y = i / kTile, x = i % kTile;
        if (r0 + y >= R || c0 + x >= C) continue;
        float mx = 0.f, my = 0.f, xx = 0.f, yy = 0.f, xy = 0.f;
#pragma unroll
        for (int k = 0; k < kWin; ++k) {
            float w = gw[k];
            mx += w * h[0][y + k][x];
            my += w * h[1][y + k][x];
            xx += w * h[2][y + k][x];
            yy += w * h[3][y + k][x];
            xy += w * h[4][y + k][x];
        }
        float sx = xx - mx * mx, sy = yy - my * my, sxy = xy - mx * my;
        float v = ((2.f * mx * my + C1) * (2.f * sxy + C2)) / ((mx * mx + my * my + C1) * (sx + sy + C2));
        s += double(v);
    }
    s = block_sum(s);
    if (tid == 0) atomicAdd(out, s);
}

// One thread per sample point of a projected tile-boundary line; marks a
// (2B+1)^2 square of the mask around its projection.
__global__ void edge_band_kernel(const tfg_rpc* __restrict__ cam, const double* __restrict__ east,
                                 const double* __restrict__ north, int grid_rows, int grid_cols, double z0,
                                 double z1, double step, uint64_t per_line, int band,
                                 uint8_t* __restrict__ mask) {
    uint64_t n_lines = uint64_t(grid_cols + 1 + grid_rows + 1) * 2;
    uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n_lines * per_line) return;
    uint64_t line = i / per_line, k = i % per_line;
    double z = (line & 1) ? z1 : z0;
    uint64_t l2 = line >> 1;
    double x, y;
    if (l2 <= uint64_t(grid_cols)) {  // x = east[l2], y along the ROI
        x = east[l2];
        y = north[0] + double(k) * step;
        if (y > north[grid_rows]) return;
    } else {
        y = north[l2 - grid_cols - 1];
        x = east[0] + double(k) * step;
        if (x > east[grid_cols]) return;
    }
    double r, c;
    if (!rpc_project(*cam, x, y, z, &r, &c)) return;
    int ir = int(floor(r)), ic = int(floor(c));
    for (int dr = -band; dr <= band; ++dr)
        for (int dc = -band; dc <= band; ++dc) {
            int rr = ir + dr, cc = ic + dc;
            if (rr >= 0 && rr < cam->image_rows && cc >= 0 && cc < cam->image_cols)
                mask[uint64_t(rr) * cam->image_cols + cc] = 1;
        }
}

} // namespace

void launch_sq_diff(const float* a, const float* b, uint64_t n, double* out, int sms, cudaStream_t st) {
    sq_diff_kernel<<<sms * 8, 256, 0, st>>>(a, b, n, out);
}
void launch_abs_diff(const float* a, const float* b, const uint8_t* mask, uint64_t n, double* out, int sms,
                     cudaStream_t st) {
    abs_diff_kernel<<<sms * 8, 256, 0, st>>>(a, b, mask, n, out);
}
void launch_ssim(const float* a, const float* b, int rows, int cols, const float* gw, double* out,
                 cudaStream_t st) {
    dim3 grid((cols - kHalo + kTile - 1) / kTile, (rows - kHalo + kTile - 1) / kTile);
    ssim_kernel<<<grid, dim3(32, 8), 0, st>>>(a, b, rows, cols, gw, out);
}
void launch_edge_band(const tfg_rpc* cam, const double* east, const double* north, int grid_rows,
                      int grid_cols, double z0, double z1, double step, uint64_t per_line, int band,
                      uint8_t* mask, cudaStream_t st) {
    uint64_t n = uint64_t(grid_cols + 1 + grid_rows + 1) * 2 * per_line;
    edge_band_kernel<<<int((n + 255) / 256), 256, 0, st>>>(cam, east, north, grid_rows, grid_cols, z0, z1,
                                                           step, per_line, band, mask);
}

} // namespace tfg
