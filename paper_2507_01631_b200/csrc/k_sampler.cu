// k_sampler.cu — K1: on-the-fly ray generation, ray/tile-box segmentation and
// per-segment stratified sampling (the paper's two custom kernels, PAPER.md:
// 320-322), bit-exact with the reference semantics.
//
// Compiled with -fmad=false: every double/float operation here rounds once,
// matching the reference's x86-64 build (see tf_common.cuh).
//
//   accept_memo_kernel + accept_solve_kernel + accept_scatter_kernel
//                    accept_rays over the window's crop union:
//                    settle memoised pixels / Newton-solve the rest / compact
//   raygen_kernel    pixel draw (rng.hpp:42-46) + ray_from_pixel (camera.cpp:105)
//                    + TileBoxSet::segments (geometry.cpp:39-48) + per-slot
//                    sample counts (sample_segments)
//   scan kernels     exclusive prefix sums (slot-bucketed sample positions)
//   tiles_kernel     128-sample single-slot work tiles for K2/K4
//   write_kernel     warp per ray: stratified samples, occupancy culling,
//                    deltas over the concatenated ray
#include <cuda_runtime.h>

#include <algorithm>

#include "tf_common.cuh"
#include "tf_kernels.h"

namespace tfg {

// ------------------------------------------------------------------ scans
// Two-kernel exclusive scan of uint32 (values and sums < 2^32): block totals,
// then per-block prefix + apply.
constexpr int kScanThreads = 512;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;

__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t v, uint32_t* total) {
    __shared__ uint32_t warp_sums[kScanThreads / 32];
    int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) warp_sums[w] = x;
    __syncthreads();
    if (w == 0) {
        uint32_t s = lane < kScanThreads / 32 ? warp_sums[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += y;
        }
        if (lane < kScanThreads / 32) warp_sums[lane] = s;
    }
    __syncthreads();
    uint32_t pre = (w > 0 ? warp_sums[w - 1] : 0) + x - v;
    if (total) *total = warp_sums[kScanThreads / 32 - 1];
    __syncthreads();
    return pre;
}

__global__ void __launch_bounds__(kScanThreads) scan_reduce_kernel(const uint32_t* __restrict__ in,
                                                                   uint64_t n,
                                                                   uint32_t* __restrict__ sums) {
    pdl_wait();
    uint64_t base = uint64_t(blockIdx.x) * kScanTile;
    uint32_t s = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        uint64_t i = base + uint64_t(threadIdx.x) * kScanItems + k;
        if (i < n) s += in[i];
    }
    uint32_t tot;
    block_exclusive_scan(s, &tot);
    if (threadIdx.x == 0) sums[blockIdx.x] = tot;
}

// Applies the block prefixes.  Each block sums the raw block totals before
// it itself (at most kScanTile of them, kScanItems per thread), so there is
// no separate pass over the block sums; the last block also writes the grand
// total.
__global__ void __launch_bounds__(kScanThreads) scan_apply_kernel(const uint32_t* __restrict__ in,
                                                                  uint64_t n,
                                                                  const uint32_t* __restrict__ sums,
                                                                  uint32_t* __restrict__ out,
                                                                  uint32_t* __restrict__ grand_total) {
    pdl_wait();
    __shared__ uint32_t s_block_pre;
    {
        uint32_t acc = 0;
        for (int j = threadIdx.x; j < int(blockIdx.x); j += blockDim.x) acc += sums[j];
        uint32_t tot;
        block_exclusive_scan(acc, &tot);
        if (threadIdx.x == 0) s_block_pre = tot;
        __syncthreads();
    }
    const uint32_t block_pre = s_block_pre;
    uint64_t base = uint64_t(blockIdx.x) * kScanTile;
    uint32_t v[kScanItems];
    uint32_t s = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        uint64_t i = base + uint64_t(threadIdx.x) * kScanItems + k;
        v[k] = i < n ? in[i] : 0;
        s += v[k];
    }
    uint32_t pre = block_exclusive_scan(s, nullptr) + block_pre;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        uint64_t i = base + uint64_t(threadIdx.x) * kScanItems + k;
        if (i < n) out[i] = pre;
        pre += v[k];
    }
    if (blockIdx.x == gridDim.x - 1 && threadIdx.x == blockDim.x - 1) {
        out[n] = pre;
        if (grand_total) *grand_total = pre;
    }
}

int scan_exclusive(const uint32_t* in, uint64_t n, uint32_t* out, uint32_t* block_sums,
                   uint32_t* grand_total, cudaStream_t st, uint64_t* launches) {
    int nb = int((n + kScanTile - 1) / kScanTile);
    if (nb < 1) nb = 1;
    if (nb > kScanTile) return 1;
    launch_pdl(scan_reduce_kernel, dim3(nb), dim3(kScanThreads), 0, st, in, n, block_sums);
    launch_pdl(scan_apply_kernel, dim3(nb), dim3(kScanThreads), 0, st, in, n, static_cast<const uint32_t*>(block_sums),
               out, grand_total);
    if (launches) *launches += 2;
    return 0;
}

// ------------------------------------------------------------------ accept list
// flag = 1 iff the candidate pixel's ray exists, hits >= 1 tile and every hit
// tile is loaded.  Two kernels: accept_memo_kernel (one light
// thread per candidate of the per-view crop-union rects) settles every pixel
// the previous window position already solved (copying its memo entry into
// this window's memo) and compacts the rest into a to-do list;
// accept_solve_kernel runs the two Newton localisations of each listed pixel
// on a lane pair, so no warp carries memo-hit lanes through a solve.
#ifndef TFG_ACCEPT_MINB
#define TFG_ACCEPT_MINB 4
#endif

__device__ __forceinline__ void candidate_pixel(const AcceptArgs& a, uint64_t idx, int* v_, int* row, int* col) {
    int v = 0;
    while (v + 1 < a.n_views && a.view_start[v + 1] <= idx) ++v;
    uint64_t local = idx - a.view_start[v];
    const int* u = a.union_rect + 4 * v;
    int ncols = u[3] - u[2];
    *v_ = v;
    *row = u[0] + int(local / uint64_t(ncols));
    *col = u[2] + int(local % uint64_t(ncols));
}

__global__ void __launch_bounds__(256) accept_memo_kernel(AcceptArgs a, uint32_t* __restrict__ flags) {
    const uint64_t idx = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    bool todo = false;
    if (idx < a.n_candidates) {
        int v, row, col;
        candidate_pixel(a, idx, &v, &row, &col);
        bool in = false;
        for (int k = 0; k < a.n_loaded; ++k) {
            const int* r = a.crop_rect + 4 * (v * kTrainSlots + k);
            if (r[0] < r[1] && row >= r[0] && row < r[1] && col >= r[2] && col < r[3]) in = true;
        }
        uint32_t info = 0;
        if (in && a.o_info) {
            // solved for the previous window position: copy its memo entry
            const int* o = a.o_rect + 4 * v;  // r0, c0, cols, rows
            if (row >= o[0] && row < o[0] + o[3] && col >= o[1] && col < o[1] + o[2]) {
                const uint64_t oi = a.o_off[v] / 3 + uint64_t(row - o[0]) * uint64_t(o[2]) + uint64_t(col - o[1]);
                info = a.o_info[oi];
                if (info & kMemoHit) {
                    const double2* src = reinterpret_cast<const double2*>(a.o_rays + 6 * oi);
                    double2* dst = reinterpret_cast<double2*>(a.m_rays + 6 * idx);
                    dst[0] = src[0];
                    dst[1] = src[1];
                    dst[2] = src[2];
                }
            }
        }
        a.m_info[idx] = info;
        if (in && !(info & kMemoDone)) {
            todo = true;
        } else {
            // outside every loaded crop, or solved for the previous window:
            // only the window test remains
            uint32_t ok = 0;
            if (info & kMemoHit) {
                int rmin = info & 127, rmax = (info >> 7) & 127, cmin = (info >> 14) & 127, cmax = (info >> 21) & 127;
                ok = (rmin >= a.win_r0 && rmax <= a.win_r1 && cmin >= a.win_c0 && cmax <= a.win_c1) ? 1u : 0u;
            }
            flags[idx] = ok;
        }
    }
    // warp-aggregated append to the to-do list
    uint32_t m = __ballot_sync(0xffffffffu, todo);
    const int lane = threadIdx.x & 31;
    uint32_t base = 0;
    if (lane == 0 && m) base = atomicAdd(a.todo_n, uint32_t(__popc(m)));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (todo) a.todo[base + __popc(m & ((1u << lane) - 1u))] = uint32_t(idx);
}

__global__ void __launch_bounds__(128, TFG_ACCEPT_MINB) accept_solve_kernel(AcceptArgs a, uint32_t* __restrict__ flags) {
    // two threads per listed pixel: one Newton localisation each (z_max / z_min)
    const uint64_t gt = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const int hi = int(gt & 1);
    const uint32_t pair = 3u << ((threadIdx.x & 31) & ~1);
    const uint32_t n_todo = *a.todo_n;
    const uint64_t stride = (uint64_t(gridDim.x) * blockDim.x) >> 1;
    for (uint64_t j = gt >> 1; j < n_todo; j += stride) {  // both lanes of a pair iterate together
        const uint64_t idx = a.todo[j];
        int v, row, col;
        candidate_pixel(a, idx, &v, &row, &col);
        uint32_t ok = 0;
        double gx = 0.0, gy = 0.0;
        int st = rpc_localize(a.cams[v], double(row), double(col), hi ? a.z_min : a.z_max, &gx, &gy,
                              a.loc ? a.loc + 2 * v + hi : nullptr);
        double ox = __shfl_xor_sync(pair, gx, 1), oy = __shfl_xor_sync(pair, gy, 1);
        int ost = __shfl_xor_sync(pair, st, 1);
        double o[3], d[3];
        uint32_t memo = kMemoDone;
        if (hi == 0 && st == 0 && ost == 0 &&
            rpc_ray_finish(gx, gy, ox, oy, a.z_min, a.z_max, o, d) == 0) {
            // candidate_tiles (tiler.cpp:70-100): XY shadow between z bounds
            double dz = d[2];
            if (dz != 0.0) {
                double ta = (a.z_max - o[2]) / dz, tb = (a.z_min - o[2]) / dz;
                if (ta > tb) { double t = ta; ta = tb; tb = t; }
                ta = (ta < 0.0) ? 0.0 : ta;  // std::max(ta, 0.0)
                if (!(tb < ta)) {
                    double ax = o[0] + ta * d[0], ay = o[1] + ta * d[1];
                    double bx = o[0] + tb * d[0], by = o[1] + tb * d[1];
                    auto cell = [](const double* e, int n, double val) {
                        // upper_bound - 1, clamped to [0, n-1]
                        int lo = 0, hi2 = n + 1;
                        while (lo < hi2) {
                            int mid = (lo + hi2) >> 1;
                            if (val < e[mid]) hi2 = mid; else lo = mid + 1;
                        }
                        int k = lo - 1;
                        return k < 0 ? 0 : (k > n - 1 ? n - 1 : k);
                    };
                    double exlo = (bx < ax) ? bx : ax, exhi = (ax < bx) ? bx : ax;
                    double nylo = (by < ay) ? by : ay, nyhi = (ay < by) ? by : ay;
                    int c0 = cell(a.east, a.grid_cols, exlo), c1 = cell(a.east, a.grid_cols, exhi);
                    int r0 = cell(a.north, a.grid_rows, nylo), r1 = cell(a.north, a.grid_rows, nyhi);
                    int hits = 0;
                    bool all_loaded = true;
                    int hr0 = 127, hr1 = 0, hc0 = 127, hc1 = 0;
                    for (int tr = r0; tr <= r1; ++tr)
                        for (int tc = c0; tc <= c1; ++tc) {
                            double box[6] = {a.east[tc],     a.north[tr],     a.z_min,
                                             a.east[tc + 1], a.north[tr + 1], a.z_max};
                            double t0, t1;
                            if (!slab(o, d, box, &t0, &t1)) continue;
                            ++hits;
                            hr0 = tr < hr0 ? tr : hr0;
                            hr1 = tr > hr1 ? tr : hr1;
                            hc0 = tc < hc0 ? tc : hc0;
                            hc1 = tc > hc1 ? tc : hc1;
                            int ti = tr * a.grid_cols + tc;
                            bool ld = false;
                            for (int k = 0; k < a.n_loaded; ++k) ld |= (a.loaded_tile[k] == ti);
                            all_loaded &= ld;
                        }
                    ok = (hits >= 1 && all_loaded) ? 1u : 0u;
                    if (hits >= 1) {
                        memo |= kMemoHit | uint32_t(hr0) | (uint32_t(hr1) << 7) | (uint32_t(hc0) << 14) |
                                (uint32_t(hc1) << 21);
                        double* pr = a.m_rays + 6 * idx;
                        pr[0] = o[0];
                        pr[1] = o[1];
                        pr[2] = o[2];
                        pr[3] = d[0];
                        pr[4] = d[1];
                        pr[5] = d[2];
                    }
                }
            }
        }
        if (hi == 0) {
            a.m_info[idx] = memo;
            flags[idx] = ok;
        }
    }
}

__global__ void accept_scatter_kernel(AcceptArgs a, const uint32_t* __restrict__ flags,
                                      const uint32_t* __restrict__ pos,
                                      uint64_t* __restrict__ out) {
    uint64_t idx = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= a.n_candidates || !flags[idx]) return;
    int v = 0;
    while (v + 1 < a.n_views && a.view_start[v + 1] <= idx) ++v;
    uint64_t local = idx - a.view_start[v];
    const int* u = a.union_rect + 4 * v;
    int ncols = u[3] - u[2];
    uint64_t row = uint64_t(u[0]) + local / uint64_t(ncols);
    uint64_t col = uint64_t(u[2]) + local % uint64_t(ncols);
    out[pos[idx]] = (uint64_t(v) << 40) | (row << 20) | col;
}

// encode_direction (nn.hpp:288-298) of the float world direction: 6 float4
__device__ __forceinline__ void write_view_encoding(const double* d, float4* ve) {
    float d3[3] = {float(d[0]), float(d[1]), float(d[2])};
    float e[24];
    int jj = 0;
    const float scales[4] = {3.14159265358979323846f, 6.28318530717958647692f,
                             12.5663706143591729538f, 25.1327412287183459077f};
    for (int f = 0; f < kViewFreqs; ++f)
        for (int c = 0; c < 3; ++c) {
            float x = scales[f] * d3[c];
            e[jj++] = sinf(x);
            e[jj++] = cosf(x);
        }
    for (int q = 0; q < 6; ++q) ve[q] = make_float4(e[4 * q], e[4 * q + 1], e[4 * q + 2], e[4 * q + 3]);
}

// ------------------------------------------------------------------ K1a
struct SegPlan {
    int nseg;
    int slot[kMaxSeg];
    double tn[kMaxSeg], tf[kMaxSeg];
    int nint[kMaxSeg];
};

// sample_segments interval counts (DESIGN.md pins): ceil(len * spm) >= 1 per
// segment; proportional rescale when the per-ray cap would be exceeded.
__device__ __forceinline__ void plan_intervals(SegPlan& p, double spm, int cap) {
    long long total = 0, sumint = 0;
    for (int k = 0; k < p.nseg; ++k) {
        double len = p.tf[k] - p.tn[k];
        long long n = (long long)ceil(len * spm);
        if (n < 1) n = 1;
        p.nint[k] = int(n);
        sumint += n;
        total += n + 1;
    }
    if (total > cap) {
        long long budget = cap - p.nseg;
        for (int k = 0; k < p.nseg; ++k) {
            long long n = (long long)p.nint[k] * budget / sumint;
            p.nint[k] = int(n < 1 ? 1 : n);
        }
    }
}

// step = (tf - tn) / n of the segment, computed once per segment by the
// caller (the same FP64 quotient for every sample of the segment)
__device__ __forceinline__ double sample_t(double tn, double tf, int n, int k, int j, bool jitter,
                                           uint64_t key, double step) {
    if (j == 0) return tn;
    if (j == n) return tf;
    float u = 0.5f;
    if (jitter) u = Rng(hash_combine(key, (uint64_t(k) << 16) | uint64_t(j))).flt();
    return tn + (double(j) + (double(u) - 0.5)) * step;
}
__device__ __forceinline__ double sample_t(const SegPlan& p, int k, int j, bool jitter,
                                           uint64_t key, double step) {
    return sample_t(p.tn[k], p.tf[k], p.nint[k], k, j, jitter, key, step);
}

__device__ __forceinline__ bool occ_test(const uint32_t* bits, float x, float y, float z) {
    int v = voxel_index(x, y, z);
    return (__ldg(bits + (v >> 5)) >> (v & 31)) & 1u;
}

// Two threads per ray: the even lane localises at z_max, the odd lane at
// z_min (the two Newton solves of ray_from_pixel are independent), the
// results are exchanged by shuffle and both lanes finish the ray with the
// same arithmetic (same bits); the interior-sample counting is split by
// sample parity; the odd lane also writes the view encoding.
#ifndef TFG_RAYGEN_MINB
#define TFG_RAYGEN_MINB 5
#endif
// kSolve = false: drawn pixels with the pixel memo only (no Newton code, so
// fewer registers and more resident warps); true: explicit pixels or no memo.
#ifndef TFG_RAYGEN_MEMO_MINB
#define TFG_RAYGEN_MEMO_MINB 8
#endif
// kLanes threads per ray: 2 for explicit pixels (one Newton localisation
// each); the memo path also runs with 8 for small batches, where the per-ray
// interior-sample loop (split over the lanes) is the latency chain.
template <bool kSolve, int kLanes>
__global__ void __launch_bounds__(128, kSolve ? TFG_RAYGEN_MINB : TFG_RAYGEN_MEMO_MINB)
    raygen_kernel(RaygenArgs a, RayRec* __restrict__ rays, float4* __restrict__ venc,
                  uint32_t* __restrict__ counts, Status* __restrict__ status) {
    static_assert(!kSolve || kLanes == 2, "the Newton path pairs two lanes per ray");
    pdl_wait();
    const int gt = blockIdx.x * blockDim.x + threadIdx.x;
    const int i = gt / kLanes, sub = gt % kLanes, hi = sub & 1;
    const uint32_t pair = 3u << ((threadIdx.x & 31) & ~1);
    const uint32_t group = ((1u << kLanes) - 1u) << ((threadIdx.x & 31) & ~(kLanes - 1));
    const bool valid = i < a.n_rays;
    const int ii = valid ? i : 0;
    uint64_t g = a.ray_begin + uint64_t(ii);
    int v, row, col;
    const double* memo = nullptr;  // the accept pass already solved accepted pixels
    if (a.pixels && a.pixel_pairs) {  // render: (row, col) pairs of the one render view
        v = 0;
        row = a.pixels[2 * ii];
        col = a.pixels[2 * ii + 1];
    } else if (a.pixels) {
        v = a.pixels[3 * ii];
        row = a.pixels[3 * ii + 1];
        col = a.pixels[3 * ii + 2];
    } else {
        uint64_t na = *a.n_accept_dev;
        Rng r(hash_combine(hash_combine(hash_combine(a.seed, kPurposePixels), a.iter), g));
        uint64_t e = na ? a.accept[r.below(na)] : 0;
        v = int(e >> 40);
        row = int((e >> 20) & 0xFFFFF);
        col = int(e & 0xFFFFF);
        if (na == 0 && valid && sub == 0) atomicOr(&status->bits, kStatusRayFail);
        if (na && a.memo_rays) {
            const int* cr = a.crop_rect + 4 * v;  // r0, c0, cols, rows: memo index = crop pixel index
            memo = a.memo_rays + 6 * (a.crop_offset[v] / 3 + uint64_t(row - cr[0]) * uint64_t(cr[2]) + uint64_t(col - cr[1]));
        }
    }
    RayRec R;
    R.view = v;
    R.row = row;
    R.col = col;
    R.target[0] = R.target[1] = R.target[2] = 0.f;
    if (memo) {
        R.status = 0;
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            R.o[q] = memo[q];
            R.d[q] = memo[3 + q];
        }
    } else if constexpr (!kSolve) {
        R.status = 1;  // empty accepted list (flagged above)
    } else {
        double gx = 0.0, gy = 0.0;
        int st = rpc_localize(a.cams[v], double(row), double(col), hi ? a.z_min : a.z_max, &gx, &gy,
                              a.loc ? a.loc + 2 * v + hi : nullptr);
        double ox = __shfl_xor_sync(pair, gx, 1), oy = __shfl_xor_sync(pair, gy, 1);
        int ost = __shfl_xor_sync(pair, st, 1);
        // status of the top (z_max) localisation first, as ray_from_pixel throws
        int st_top = hi ? ost : st, st_bot = hi ? st : ost;
        R.status = st_top ? st_top : st_bot;
        if (R.status == 0) {
            double tx = hi ? ox : gx, ty = hi ? oy : gy, bx = hi ? gx : ox, by = hi ? gy : oy;
            R.status = rpc_ray_finish(tx, ty, bx, by, a.z_min, a.z_max, R.o, R.d);
        }
    }
    if (valid && sub == 0)
        for (int s = 0; s < a.slots.n; ++s) counts[uint64_t(s) * a.n_rays + i] = 0;
    R.nseg = 0;
    if (R.status != 0) {
        if (valid && sub == 0) {
            atomicOr(&status->bits, kStatusRayFail);
            rays[i] = R;
        }
        return;
    }
    if (a.crop_bytes && sub == 0) {
        const int* cr = a.crop_rect + 4 * v;  // r0, c0, cols, rows
        const uint8_t* px = a.crop_bytes + a.crop_offset[v] +
                            3 * (uint64_t(row - cr[0]) * uint64_t(cr[2]) + uint64_t(col - cr[1]));
        for (int c = 0; c < 3; ++c) R.target[c] = float(px[c]) / 255.0f;  // u8_to_unit
    }
    // TileBoxSet::segments: hits in slot order, stable insertion sort on t_near
    SegPlan p;
    p.nseg = 0;
    bool overflow = false;
    for (int s = 0; s < a.slots.n; ++s) {
        double t0, t1;
        double box[6];  // from the kernel parameters by value (a pointer into them would copy the block to local memory)
#pragma unroll
        for (int q = 0; q < 6; ++q) box[q] = a.slots.box[s][q];
        if (!slab(R.o, R.d, box, &t0, &t1)) continue;
        if (p.nseg == kMaxSeg) {
            overflow = true;
            break;
        }
        int j = p.nseg++;
        while (j > 0 && t0 < p.tn[j - 1]) {
            p.tn[j] = p.tn[j - 1];
            p.tf[j] = p.tf[j - 1];
            p.slot[j] = p.slot[j - 1];
            --j;
        }
        p.tn[j] = t0;
        p.tf[j] = t1;
        p.slot[j] = s;
    }
    if (overflow && valid && sub == 0) atomicOr(&status->bits, kStatusSegOverflow);
    plan_intervals(p, a.spm, a.cap);
    uint64_t key = hash_combine(hash_combine(hash_combine(a.seed, kPurposeJitter), a.iter), g);
    R.nseg = p.nseg;
    const double o0 = R.o[0], o1 = R.o[1], o2 = R.o[2], d0 = R.d[0], d1 = R.d[1], d2 = R.d[2];
    for (int k = 0; k < p.nseg; ++k) {
        // slot frame values from the kernel parameters (no pointer into them,
        // which would copy the parameter block to local memory)
        const int sl = p.slot[k];
        const double f0 = a.slots.frame[sl][0], f1 = a.slots.frame[sl][1], f2 = a.slots.frame[sl][2];
        const double f3 = a.slots.frame[sl][3], f4 = a.slots.frame[sl][4], f5 = a.slots.frame[sl][5];
        const uint32_t* bits = a.occ_bits[sl];
        const int n = p.nint[k];
        const double tn = p.tn[k], tf = p.tf[k];
        const double step = (tf - tn) / n;
        int cnt = 0;
        for (int j = 1 + sub; j < n; j += kLanes) {
            double t = sample_t(tn, tf, n, k, j, a.jitter, key, step);
            float lx = float((o0 + t * d0 - f0) * f3);
            float ly = float((o1 + t * d1 - f1) * f4);
            float lz = float((o2 + t * d2 - f2) * f5);
            cnt += occ_test(bits, lx, ly, lz);
        }
#pragma unroll
        for (int o = 1; o < kLanes; o <<= 1) cnt += __shfl_xor_sync(group, cnt, o);
        cnt += 2;  // endpoints are never culled
        R.slot[k] = uint8_t(p.slot[k]);
        R.tn[k] = p.tn[k];
        R.tf[k] = p.tf[k];
        R.nint[k] = uint16_t(n);
        R.cnt[k] = uint16_t(cnt);
        if (valid && sub == 0) counts[uint64_t(p.slot[k]) * a.n_rays + i] = uint32_t(cnt);
    }
    if (!valid) return;
    if (sub == 0) {
        rays[i] = R;
        return;
    }
    if (sub == 1) write_view_encoding(R.d, venc + uint64_t(i) * 6);
}

// Slot buckets -> 128-sample single-slot tiles (one block).
__global__ void tiles_kernel(const uint32_t* __restrict__ P, int n_rays, int nslots,
                             uint64_t capacity, int max_tiles, TileDesc* __restrict__ tiles,
                             Status* __restrict__ status) {
    pdl_wait();
    // every CTA derives the slot buckets' tile bases from P (a few loads);
    // block 0 publishes the totals, all CTAs write their share of the tiles
    __shared__ uint32_t tile_base[kMaxSlots + 1], bucket[kMaxSlots + 1];
    __shared__ int ok;
    if (threadIdx.x == 0) {
        uint32_t tb = 0;
        for (int s = 0; s <= nslots; ++s) bucket[s] = P[uint64_t(s) * n_rays];
        for (int s = 0; s < nslots; ++s) {
            tile_base[s] = tb;
            tb += (bucket[s + 1] - bucket[s] + 127) / 128;
        }
        tile_base[nslots] = tb;
        const uint64_t total = bucket[nslots];
        ok = !(total > capacity || int(tb) > max_tiles);
        if (blockIdx.x == 0) {
            status->n_samples = total;
            status->n_tiles = ok ? tb : 0;
            if (!ok) atomicOr(&status->bits, kStatusSampleOverflow);
        }
    }
    __syncthreads();
    if (!ok) return;
    const uint32_t n_tiles = tile_base[nslots];
    for (uint32_t g = blockIdx.x * blockDim.x + threadIdx.x; g < n_tiles; g += gridDim.x * blockDim.x) {
        int s = 0;
        while (s + 1 < nslots && g >= tile_base[s + 1]) ++s;
        TileDesc d;
        d.start = bucket[s] + 128 * (g - tile_base[s]);
        const uint32_t rem = bucket[s + 1] - d.start;
        d.n = uint16_t(rem < 128 ? rem : 128);
        d.slot = uint16_t(s);
        tiles[g] = d;
    }
}

// ------------------------------------------------------------------ K1c
// Warp per ray: regenerate the stratified samples of every segment, cull
// interior samples in clear occupancy voxels (ballot compaction), write them
// to the ray's slot buckets, and delta = t_next - t over the concatenated ray
// (double, then rounded; duplicate boundary samples get delta = 0); the last
// kept sample's delta is the remaining distance to the z_min exit capped at
// delta_cap.
#ifndef TFG_WRITE_THREADS
#define TFG_WRITE_THREADS 128
#endif
#ifndef TFG_WRITE_MINB
#define TFG_WRITE_MINB 8  // 64 registers, no spills: 8 us faster than the unbounded 80
#endif
// Lane q < 16 of the ray's warp writes word q of its composite header.
__device__ __forceinline__ void write_hdr(RayHdr* __restrict__ hdr, const RayRec& R, const uint32_t* __restrict__ P,
                                          int n_rays, int i, int lane) {
    const int nseg = R.status == 0 ? R.nseg : -1;
    uint32_t w = 0;
    if (lane < kMaxSeg) {
        w = lane < nseg ? P[uint64_t(R.slot[lane]) * n_rays + i] : 0u;
    } else if (lane < kMaxSeg + kMaxSeg / 2) {
        const int k = 2 * (lane - kMaxSeg);
        w = (k < nseg ? uint32_t(R.cnt[k]) : 0u) | ((k + 1 < nseg ? uint32_t(R.cnt[k + 1]) : 0u) << 16);
    } else if (lane < kMaxSeg + kMaxSeg / 2 + 3) {
        w = __float_as_uint(R.target[lane - kMaxSeg - kMaxSeg / 2]);
    } else if (lane == 15) {
        w = uint32_t(nseg);
    }
    if (lane < 16) reinterpret_cast<uint32_t*>(hdr + i)[lane] = w;
}

__global__ void __launch_bounds__(TFG_WRITE_THREADS, TFG_WRITE_MINB) write_kernel(RaygenArgs a, const RayRec* __restrict__ rays,
                                                    const uint32_t* __restrict__ P,
                                                    const Status* __restrict__ status,
                                                    SampleArrays out, RayHdr* __restrict__ hdr) {
    pdl_wait();
    int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    int lane = threadIdx.x & 31;
    if (warp >= a.n_rays) return;
    if (status->bits & kStatusSampleOverflow) return;
    const RayRec& R = rays[warp];
    if (R.status != 0) {
        write_hdr(hdr, R, P, a.n_rays, warp, lane);
        return;
    }
    uint64_t g = a.ray_begin + uint64_t(warp);
    uint64_t key = hash_combine(hash_combine(hash_combine(a.seed, kPurposeJitter), a.iter), g);
    // segment fields straight from the (warp-uniform) ray record and the
    // slot frame from the kernel parameters: no local-memory copies
    const int nseg = R.nseg;
    const double o0 = R.o[0], o1 = R.o[1], o2 = R.o[2], d0 = R.d[0], d1 = R.d[1], d2 = R.d[2];
    const uint32_t lt = (1u << lane) - 1u;
    long long pend_pos = -1;
    double pend_t = 0.0;
    for (int k = 0; k < nseg; ++k) {
        const int s = R.slot[k];
        const double f0 = a.slots.frame[s][0], f1 = a.slots.frame[s][1], f2 = a.slots.frame[s][2];
        const double f3 = a.slots.frame[s][3], f4 = a.slots.frame[s][4], f5 = a.slots.frame[s][5];
        const uint32_t* bits = a.occ_bits[s];
        uint64_t base = P[uint64_t(s) * a.n_rays + warp];
        uint32_t written = 0;
        const int n = R.nint[k];
        const double tn = R.tn[k], tf = R.tf[k];
        const double step = (tf - tn) / n;
        for (int j0 = 0; j0 <= n; j0 += 32) {
            int j = j0 + lane;
            bool valid = j <= n;
            double t = 0.0;
            float lx = 0.f, ly = 0.f, lz = 0.f;
            bool endp = (j == 0 || j == n);
            bool keep = false;
            if (valid) {
                t = sample_t(tn, tf, n, k, j, a.jitter, key, step);
                lx = float((o0 + t * d0 - f0) * f3);
                ly = float((o1 + t * d1 - f1) * f4);
                lz = float((o2 + t * d2 - f2) * f5);
                keep = endp || occ_test(bits, lx, ly, lz);
            }
            uint32_t mask = __ballot_sync(0xffffffffu, keep);
            if (mask == 0u) continue;
            int first = __ffs(mask) - 1;
            int last = 31 - __clz(mask);
            double t_first = __shfl_sync(0xffffffffu, t, first);
            if (lane == 0 && pend_pos >= 0)
                out.td[pend_pos] = make_float2(float(pend_t), float(t_first - pend_t));
            uint32_t gt = mask & ~(lt | (1u << lane));
            int nxt = gt ? (__ffs(gt) - 1) : lane;
            double t_next = __shfl_sync(0xffffffffu, t, nxt);
            if (keep) {
                uint64_t pos = base + written + __popc(mask & lt);
                out.local[pos] = make_float4(lx, ly, lz, __int_as_float(warp));
                // the chunk's last kept sample is completed once its successor is known
                if (gt) out.td[pos] = make_float2(float(t), float(t_next - t));
                out.endpoint[pos] = endp ? 1 : 0;
            }
            uint32_t kept = __popc(mask);
            pend_pos = (long long)(base + written + kept - 1);
            pend_t = __shfl_sync(0xffffffffu, t, last);
            written += kept;
        }
    }
    if (lane == 0 && pend_pos >= 0) {
        double texit = (a.z_min - o2) / d2;
        double r = texit - pend_t;
        if (r < 0) r = 0;
        if (r > a.delta_cap) r = a.delta_cap;
        out.td[pend_pos] = make_float2(float(pend_t), float(r));
    }
    write_hdr(hdr, R, P, a.n_rays, warp, lane);  // last: off the samples' critical path
}

// ------------------------------------------------------------------ batch import
// A caller-built RaySegmentBatch (tfg_batch_import; the forward_batch /
// backward_batch drop-in) into the device batch layout the sampler writes:
// per ray its runs of same-slot samples become the ray's segments (a ray
// crosses each convex tile box at most once, so at most one run per slot),
// per-slot counts -> exclusive scan -> slot buckets -> 128-sample tiles.
__global__ void __launch_bounds__(128) import_plan_kernel(ImportArgs a, RayRec* __restrict__ rays,
                                                          float4* __restrict__ venc, uint32_t* __restrict__ counts,
                                                          Status* __restrict__ status) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= a.n_rays) return;
    const tfg_ray_entry& E = a.rays[i];
    RayRec R;
    for (int q = 0; q < 3; ++q) {
        R.o[q] = E.origin[q];
        R.d[q] = E.direction[q];
        R.target[q] = E.target[q];
    }
    R.view = E.image_id;
    R.row = E.row;
    R.col = E.col;
    R.status = 0;
    R.nseg = 0;
    for (int s = 0; s < a.nslots; ++s) counts[uint64_t(s) * a.n_rays + i] = 0;
    const uint32_t q0 = a.offsets[i], q1 = a.offsets[i + 1];
    uint32_t seen = 0;
    bool bad = q1 < q0;
    for (uint32_t q = q0; q < q1 && !bad;) {
        const int s = a.slot[q];
        uint32_t e = q + 1;
        while (e < q1 && a.slot[e] == s) ++e;
        if (s >= a.nslots || (seen >> s) & 1u || R.nseg == kMaxSeg) {
            bad = true;
            break;
        }
        seen |= 1u << s;
        const int k = R.nseg++;
        R.slot[k] = uint8_t(s);
        R.cnt[k] = uint16_t(e - q);
        R.nint[k] = uint16_t(e - q - 1);
        R.tn[k] = a.t[q];
        R.tf[k] = a.t[e - 1];
        counts[uint64_t(s) * a.n_rays + i] = e - q;
        q = e;
    }
    if (bad) {
        atomicOr(&status->bits, kStatusBadBatch);
        R.status = 2;
        R.nseg = 0;
        for (int s = 0; s < a.nslots; ++s) counts[uint64_t(s) * a.n_rays + i] = 0;
    }
    rays[i] = R;
    write_view_encoding(R.d, venc + uint64_t(i) * 6);
}

__global__ void __launch_bounds__(128) import_scatter_kernel(ImportArgs a, const RayRec* __restrict__ rays,
                                                             const uint32_t* __restrict__ P,
                                                             const Status* __restrict__ status, SampleArrays out,
                                                             RayHdr* __restrict__ hdr) {
    pdl_wait();
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (warp >= a.n_rays || (status->bits & kStatusSampleOverflow)) return;
    const RayRec& R = rays[warp];
    write_hdr(hdr, R, P, a.n_rays, warp, lane);
    if (R.status != 0) return;
    uint32_t q = a.offsets[warp];
    for (int k = 0; k < R.nseg; ++k) {
        const uint64_t base = P[uint64_t(R.slot[k]) * a.n_rays + warp];
        const int n = R.cnt[k];
        for (int j = lane; j < n; j += 32) {
            const uint32_t s = q + j;
            out.local[base + j] = make_float4(a.local[3 * uint64_t(s)], a.local[3 * uint64_t(s) + 1],
                                              a.local[3 * uint64_t(s) + 2], __int_as_float(warp));
            out.td[base + j] = make_float2(a.t[s], a.delta[s]);
            out.endpoint[base + j] = a.endpoint[s];
        }
        q += n;
    }
}

int launch_import(const ImportArgs& a, RayRec* rays, RayHdr* hdr, float4* venc, uint32_t* counts, uint32_t* P,
                  uint32_t* block_sums, TileDesc* tiles, int max_tiles, SampleArrays out, uint64_t capacity,
                  Status* status, cudaStream_t st, uint64_t* launches) {
    import_plan_kernel<<<(a.n_rays + 127) / 128, 128, 0, st>>>(a, rays, venc, counts, status);
    uint64_t n = uint64_t(a.nslots) * a.n_rays;
    if (scan_exclusive(counts, n, P, block_sums, nullptr, st, launches)) return 1;
    launch_pdl(tiles_kernel, dim3(std::max(1, std::min(148, (max_tiles + 255) / 256))), dim3(256), 0, st, P, a.n_rays,
               a.nslots, capacity, max_tiles, tiles, status);
    launch_pdl(import_scatter_kernel, dim3((a.n_rays * 32 + 127) / 128), dim3(128), 0, st, a,
               static_cast<const RayRec*>(rays), static_cast<const uint32_t*>(P), static_cast<const Status*>(status),
               out, hdr);
    *launches += 3;
    return 0;
}

// ------------------------------------------------------------------ host launchers
int launch_accept(const AcceptArgs& args, uint32_t* flags, uint32_t* pos, uint32_t* block_sums,
                  uint32_t* n_out, uint64_t* out, cudaStream_t st, uint64_t* launches) {
    AcceptArgs a = args;
    a.todo = pos;
    if (a.n_candidates == 0) {
        if (n_out) cudaMemsetAsync(n_out, 0, 4, st);
        return 0;
    }
    int nb = int((a.n_candidates + 127) / 128);
    cudaMemsetAsync(a.todo_n, 0, 4, st);
    accept_memo_kernel<<<int((a.n_candidates + 255) / 256), 256, 0, st>>>(a, flags);
    // one lane pair per candidate (the to-do list is at most that long; pairs
    // past its end leave at once): measured faster than a persistent grid
    uint64_t solve_blocks = (2 * a.n_candidates + 127) / 128;
    accept_solve_kernel<<<int(solve_blocks), 128, 0, st>>>(a, flags);
    if (scan_exclusive(flags, a.n_candidates, pos, block_sums, n_out, st, launches)) return 1;
    accept_scatter_kernel<<<nb, 128, 0, st>>>(a, flags, pos, out);
    *launches += 3;
    return 0;
}

__global__ void loc_start_kernel(const tfg_rpc* __restrict__ cams, int n, double z_min, double z_max,
                                 LocStart* __restrict__ out) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t < 2 * n) rpc_loc_start(cams[t >> 1], (t & 1) ? z_min : z_max, out + t);
}

void launch_loc_start(const tfg_rpc* cams, int n, double z_min, double z_max, LocStart* out, cudaStream_t st) {
    if (n > 0) loc_start_kernel<<<(2 * n + 63) / 64, 64, 0, st>>>(cams, n, z_min, z_max, out);
}

int launch_sampler(const RaygenArgs& a, RayRec* rays, RayHdr* hdr, float4* venc, uint32_t* counts,
                   uint32_t* P, uint32_t* block_sums, TileDesc* tiles, int max_tiles,
                   SampleArrays out, uint64_t capacity, Status* status, cudaStream_t st,
                   uint64_t* launches) {
#ifndef TFG_RAYGEN_WIDE_BELOW
#define TFG_RAYGEN_WIDE_BELOW 32768  // memo draws of fewer rays: 8 lanes per ray
#endif
    if (!a.pixels && a.memo_rays && a.n_rays < TFG_RAYGEN_WIDE_BELOW)
        launch_pdl(raygen_kernel<false, 8>, dim3((8 * a.n_rays + 127) / 128), dim3(128), 0, st, a, rays, venc,
                   counts, status);
#ifndef TFG_RAYGEN_LANES
#define TFG_RAYGEN_LANES 2  // memo draws of TFG_RAYGEN_WIDE_BELOW rays or more
#endif
    else if (!a.pixels && a.memo_rays)
        launch_pdl(raygen_kernel<false, TFG_RAYGEN_LANES>, dim3((TFG_RAYGEN_LANES * a.n_rays + 127) / 128), dim3(128),
                   0, st, a, rays, venc, counts, status);
    else
        launch_pdl(raygen_kernel<true, 2>, dim3((2 * a.n_rays + 127) / 128), dim3(128), 0, st, a, rays, venc,
                   counts, status);
    uint64_t n = uint64_t(a.slots.n) * a.n_rays;
    if (scan_exclusive(counts, n, P, block_sums, nullptr, st, launches)) return 1;
    launch_pdl(tiles_kernel, dim3(std::max(1, std::min(148, (max_tiles + 255) / 256))), dim3(256), 0, st, P, a.n_rays, a.slots.n,
               capacity, max_tiles, tiles, status);
    launch_pdl(write_kernel, dim3((a.n_rays * 32 + TFG_WRITE_THREADS - 1) / TFG_WRITE_THREADS), dim3(TFG_WRITE_THREADS), 0,
               st, a, rays, P, status, out, hdr);
    *launches += 3;
    return 0;
}

} // namespace tfg
