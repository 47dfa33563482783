// k_composite.cu — K3: front-to-back volume compositing over the concatenated
// segments of each ray (transmittance carried across tiles),
// the colour loss (channel-mean convention of the example at
// :377) and the analytic render backward:
//   alpha_k = 1 - exp(-sigma_k delta_k),  T_k = prod_{j<k} (1 - alpha_j),
//   w_k = T_k alpha_k,  C = sum w_k c_k + T_N bg,
//   dC/dc_k = w_k,  dC/dsigma_k = delta_k (T_{k+1} c_k - R_k),
//   R_k = sum_{j>k} w_j c_j + T_N bg = (C - T_N bg - P_k) + T_N bg,
// with P_k the inclusive prefix of w c; the backward only needs g . R_k, so
// it scans the scalar w (g . c) once instead of three channels.  One warp per
// ray at a time (persistent warps; the next ray's header is loaded during the
// current ray); samples are read segment by segment from their slot buckets
// (coalesced runs), transmittance is a warp product scan with a carried
// prefix.  Memory-bound.
#include <cuda_runtime.h>

#include <algorithm>

#include "tf_common.cuh"
#include "tf_kernels.h"

namespace tfg {

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// The batch loss is summed without same-address global atomics (65,536 of
// them, serialised in L2, cost a third of the kernel): each block sums its
// rays in smem, the last warp to arrive stores the block's partial, and
// loss_reduce_kernel adds the partials.  Every warp arrives exactly once.
__device__ __forceinline__ void loss_arrive(double* blk_sum, unsigned* blk_n, double* parts, double term,
                                            int lane) {
    if (lane != 0) return;
    if (term != 0.0) atomicAdd(blk_sum, term);
    __threadfence_block();
    if (atomicAdd(blk_n, 1u) == (blockDim.x >> 5) - 1) {
        __threadfence_block();
        parts[blockIdx.x] = *reinterpret_cast<volatile double*>(blk_sum);
    }
}

__global__ void __launch_bounds__(1024) loss_reduce_kernel(const double* __restrict__ parts, int n,
                                                           Status* __restrict__ status) {
    __shared__ double w[32];
    pdl_wait();
    double v = 0.0;
    for (int k = threadIdx.x; k < n; k += blockDim.x) v += parts[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) w[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x < 32) {
        v = threadIdx.x < (blockDim.x >> 5) ? w[threadIdx.x] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (threadIdx.x == 0) status->loss += v;
    }
}

#ifndef TFG_COMPOSITE_THREADS
#define TFG_COMPOSITE_THREADS 256  // >= 256: d_loss_parts holds max_rays / 8 block partials
#endif
// 2 cached chunks at 4 CTAs/SM (64 registers): measured 0.087 ms against
// 0.090 (3 chunks, 4 CTAs/SM) and 0.100 (4 chunks, 3 CTAs/SM)
#ifndef TFG_COMPOSITE_MINB
#define TFG_COMPOSITE_MINB 4
#endif
#ifndef TFG_COMPOSITE_CACHE
#define TFG_COMPOSITE_CACHE 2
#endif
__global__ void __launch_bounds__(TFG_COMPOSITE_THREADS, TFG_COMPOSITE_MINB) composite_kernel(CompositeArgs a) {
    __shared__ double blk_sum;
    __shared__ unsigned blk_n;
    const int lane = threadIdx.x & 31;
    const int warp0 = int((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    const int nwarps = int((gridDim.x * blockDim.x) >> 5);
    if (threadIdx.x == 0) {
        blk_sum = 0.0;
        blk_n = 0u;
    }
    __syncthreads();
    pdl_wait();  // the forward's sigma/rgb
    const bool run = !(a.status_in->bits & kStatusSampleOverflow);
    double loss = 0.0;  // this warp's rays (lane 0)
    // Persistent warps, one ray at a time: the next ray's 64 B header is
    // loaded (one word per lane 0-15) while this ray is composited, so a ray
    // starts with its sample loads instead of a dependent header load.
    uint32_t hw_next = 0;
    if (run && warp0 < a.n_rays && lane < 16) hw_next = __ldg(reinterpret_cast<const uint32_t*>(a.hdr + warp0) + lane);
    for (int i = warp0; run && i < a.n_rays; i += nwarps) {
        const uint32_t hw = hw_next;
        if (i + nwarps < a.n_rays && lane < 16)
            hw_next = __ldg(reinterpret_cast<const uint32_t*>(a.hdr + i + nwarps) + lane);
        // the ray's segments from its header, held in registers: bucket position
        // and kept count per segment, their prefix sums for locating a sample of
        // the concatenated ray
        const int hseg = int(__shfl_sync(0xffffffffu, hw, 15));
        const bool ray_ok = hseg >= 0;
        const int nseg = ray_ok ? hseg : 0;
        uint32_t base[kMaxSeg], cwd[4];
#pragma unroll
        for (int k = 0; k < kMaxSeg; ++k) base[k] = __shfl_sync(0xffffffffu, hw, k);
#pragma unroll
        for (int k = 0; k < 4; ++k) cwd[k] = __shfl_sync(0xffffffffu, hw, 8 + k);
        float target[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) target[c] = __uint_as_float(__shfl_sync(0xffffffffu, hw, 12 + c));
        int pre[kMaxSeg + 1];  // pre[k]: samples of the ray before segment k
        pre[0] = 0;
#pragma unroll
        for (int k = 0; k < kMaxSeg; ++k) {
            const int c = k < nseg ? int((cwd[k >> 1] >> (16 * (k & 1))) & 0xffffu) : 0;
            pre[k + 1] = pre[k] + c;
        }
        const int m = pre[kMaxSeg];
        const uint32_t FULL = 0xffffffffu;
        // The first kCache chunks of 32 samples stay in registers between the
        // forward and the backward sweep (rays have ~70 samples), longer rays
        // re-read their tail.
        constexpr int kCache = TFG_COMPOSITE_CACHE;
        float4 cio[kCache];
        float2 ctd[kCache];
        uint64_t cpos[kCache];
        float cw[kCache], ct1[kCache];  // weight w_k and T_{k+1} of the cached samples
        // (base / pre captured by value: a by-reference capture would put them in local memory)
        auto fetch = [base, pre, m, &a](int q, float4& io, float2& td, uint64_t& pos) {
            io = make_float4(0.f, 0.f, 0.f, 0.f);
            td = make_float2(0.f, 0.f);
            pos = 0;
            if (q < m) {
                // segment of sample q: unrolled selects (no local-memory arrays)
                uint32_t b = base[0];
                int p0 = 0;
#pragma unroll
                for (int k = 1; k < kMaxSeg; ++k)
                    if (q >= pre[k]) {
                        b = base[k];
                        p0 = pre[k];
                    }
                pos = uint64_t(b) + (q - p0);
                io = a.s.io[pos];
                td = a.s.td[pos];
            }
        };
        // ---------------- forward
        float T = 1.f, cr = 0.f, cg = 0.f, cb = 0.f, dep = 0.f, op = 0.f;
        float w_last = 0.f, t1_last = 0.f;  // of the lane's sample in the last chunk processed
        auto fwd_chunk = [&](const float4& io, const float2& td) {
            float alpha = 1.f - expf(-(io.x * td.y));
            float keep = 1.f - alpha;
            float incl = keep;  // inclusive product scan of (1 - alpha)
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                float y = __shfl_up_sync(FULL, incl, o);
                if (lane >= o) incl *= y;
            }
            float excl = __shfl_up_sync(FULL, incl, 1);
            if (lane == 0) excl = 1.f;
            float w = T * excl * alpha;
            cr += w * io.y;
            cg += w * io.z;
            cb += w * io.w;
            dep += w * td.x;
            op += w;
            w_last = w;
            t1_last = T * incl;
            T *= __shfl_sync(FULL, incl, 31);
        };
#pragma unroll
        for (int ci = 0; ci < kCache; ++ci) {
            if (ci * 32 < m) {
                fetch(ci * 32 + lane, cio[ci], ctd[ci], cpos[ci]);
                fwd_chunk(cio[ci], ctd[ci]);
                cw[ci] = w_last;
                ct1[ci] = t1_last;
            }
        }
        const float T_after_cache = T;
        for (int q0 = kCache * 32; q0 < m; q0 += 32) {
            float4 io;
            float2 td;
            uint64_t pos;
            fetch(q0 + lane, io, td, pos);
            fwd_chunk(io, td);
        }
        cr = warp_sum(cr);
        cg = warp_sum(cg);
        cb = warp_sum(cb);
        dep = warp_sum(dep);
        op = warp_sum(op);
        float rr = cr + T * a.bg.x, rg = cg + T * a.bg.y, rb = cb + T * a.bg.z;
        if (lane == 0) {
            if (a.ray_rgb) {
                a.ray_rgb[3 * i] = rr;
                a.ray_rgb[3 * i + 1] = rg;
                a.ray_rgb[3 * i + 2] = rb;
            }
            if (a.ray_depth) a.ray_depth[i] = dep / fmaxf(op, 1e-10f);
            if (a.ray_opacity) a.ray_opacity[i] = op;
        }
        if (!a.backward || !ray_ok) continue;
        float er = rr - target[0], eg = rg - target[1], eb = rb - target[2];
        loss += double(er * er + eg * eg + eb * eb);
        float gr = 2.f * er * a.inv3b, gg = 2.f * eg * a.inv3b, gb = 2.f * eb * a.inv3b;
        // ---------------- backward
        // g . R_k = g . Cfg - P_k + T_N (g . bg), with P_k the inclusive prefix of
        // the scalar w_j (g . c_j): one scan instead of one per channel
        float T2 = 1.f, ps = 0.f;
        const float gC = (gr * cr + gg * cg) + gb * cb;
        const float gBg = T * ((gr * a.bg.x + gg * a.bg.y) + gb * a.bg.z);    // w and T_{k+1} of a chunk: recomputed exactly as the forward sweep did
        // (same operations, same order), or taken from the forward's cache
        auto chunk_weights = [&](const float4& io, const float2& td, float& w, float& Tk1) {
            float alpha = 1.f - expf(-(io.x * td.y));
            float keep = 1.f - alpha;
            float incl = keep;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                float y = __shfl_up_sync(FULL, incl, o);
                if (lane >= o) incl *= y;
            }
            float excl = __shfl_up_sync(FULL, incl, 1);
            if (lane == 0) excl = 1.f;
            w = T2 * excl * alpha;
            Tk1 = T2 * incl;
            T2 *= __shfl_sync(FULL, incl, 31);
        };
        auto bwd_chunk = [&](int q, const float4& io, const float2& td, uint64_t pos, float w, float Tk1) {
            float sg = io.x, de = td.y;
            const float gc = (gr * io.y + gg * io.z) + gb * io.w;  // g . c_k
            float sc = w * gc;  // inclusive prefix of w (g . c)
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                float y = __shfl_up_sync(FULL, sc, o);
                if (lane >= o) sc += y;
            }
            const float gR = (gC - (ps + sc)) + gBg;  // g . R_k
            float ds = de * (Tk1 * gc - gR);
            if (q < m) {
                // pre-activation gradients for K4: d raw = dsigma * exp'(raw)
                // (= sigma, or 0 where the activation is clamped, nn.hpp:270-280),
                // d pre-sigmoid = dc * s (1 - s) (nn.hpp:283-285)
                float dr = w * gr, dg = w * gg, db = w * gb;
                float draw = sg >= a.density_max ? 0.f : ds * sg;
                a.s.io[pos] = make_float4(draw, dr * io.y * (1.f - io.y), dg * io.z * (1.f - io.z),
                                          db * io.w * (1.f - io.w));
                if (a.export_io) a.export_io[pos] = make_float4(ds, dr, dg, db);
            }
            ps += __shfl_sync(FULL, sc, 31);
        };
#pragma unroll
        for (int ci = 0; ci < kCache; ++ci)
            if (ci * 32 < m) bwd_chunk(ci * 32 + lane, cio[ci], ctd[ci], cpos[ci], cw[ci], ct1[ci]);
        T2 = T_after_cache;  // the uncached tail continues from the forward's transmittance
        for (int q0 = kCache * 32; q0 < m; q0 += 32) {
            float4 io;
            float2 td;
            uint64_t pos;
            fetch(q0 + lane, io, td, pos);
            float w, Tk1;
            chunk_weights(io, td, w, Tk1);
            bwd_chunk(q0 + lane, io, td, pos, w, Tk1);
        }
    }
    loss_arrive(&blk_sum, &blk_n, a.loss_parts, loss, lane);
}

void launch_composite(const CompositeArgs& a, cudaStream_t st, uint64_t* launches) {
#ifndef TFG_COMPOSITE_WAVES
#define TFG_COMPOSITE_WAVES 1  // resident blocks per SM x this = the persistent grid
#endif
    const int need = (a.n_rays * 32 + TFG_COMPOSITE_THREADS - 1) / TFG_COMPOSITE_THREADS;
    const int sms = a.sms > 0 ? a.sms : 148;
    const int blocks = std::max(1, std::min(need, sms * TFG_COMPOSITE_MINB * TFG_COMPOSITE_WAVES));
    launch_pdl(composite_kernel, dim3(blocks), dim3(TFG_COMPOSITE_THREADS), 0, st, a);
    *launches += 1;
    if (a.backward) {
        launch_pdl(loss_reduce_kernel, dim3(1), dim3(1024), 0, st, static_cast<const double*>(a.loss_parts), blocks,
                   a.status);
        *launches += 1;
    }
}

} // namespace tfg
