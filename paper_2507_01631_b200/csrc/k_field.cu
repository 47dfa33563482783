// k_field.cu — K2/K4: per-tile NeRF field forward / backward, and K6 the
// occupancy update.  Replaces forward_batch / backward_batch (field.hpp:
// 185-197; MlpT nn.hpp:90-157, HashGridT nn.hpp:213-245) and
// TileField::update_occupancy (field.hpp:100-102).
//
// Work unit: a tile of <= 128 consecutive samples of ONE slot bucket (built
// by K1), so the density MLP of a tile uses a single tile's weights.  Blocks
// are persistent (grid = SMs x resident blocks) and walk the tile list read
// from device memory (no host sync between K1 and K2/K4).
//
// This translation unit is the CUDA-core reference implementation of the
// field math (FP32 FFMA); k_field_tc.cu holds the tcgen05/TMEM path.
#include <cuda_runtime.h>

#include "tf_common.cuh"
#include "tf_hash.cuh"
#include "tf_kernels.h"

namespace tfg {

constexpr int kTile = 128;

__device__ __forceinline__ float sigmoidf_(float x) { return 1.f / (1.f + expf(-x)); }

// ------------------------------------------------------------------ K2 forward
// smem: density weights of the current slot (2128) + colour weights (6915).
constexpr int kFwdSmemFloats = kDnetParams + kColorParams + 1;

__device__ __forceinline__ void load_floats(float* dst, const float* __restrict__ src, int n) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];
}

__device__ __forceinline__ void field_point_fwd(const float* __restrict__ Wd,
                                                const float* __restrict__ Wc, const float* feat,
                                                const float4* __restrict__ ve, float lim,
                                                float dmax, float* sigma, float* rgb) {
    float h[kDHidden];
#pragma unroll
    for (int o = 0; o < kDHidden; ++o) {
        float acc = Wd[kDB1 + o];
#pragma unroll
        for (int i = 0; i < kFeatDim; ++i) acc += Wd[kDW1 + o * kFeatDim + i] * feat[i];
        h[o] = acc < 0.f ? 0.f : acc;
    }
    float cin[kCIn + 1];
#pragma unroll
    for (int o = 0; o < kDOut; ++o) {
        float acc = Wd[kDB2 + o];
#pragma unroll
        for (int i = 0; i < kDHidden; ++i) acc += Wd[kDW2 + o * kDHidden + i] * h[i];
        if (o == 0) {
            *sigma = acc >= lim ? dmax : expf(acc);
        } else {
            cin[o - 1] = acc;
        }
    }
#pragma unroll
    for (int q = 0; q < 6; ++q) {
        float4 e = __ldg(ve + q);
        cin[kEmb + 4 * q] = e.x;
        cin[kEmb + 4 * q + 1] = e.y;
        cin[kEmb + 4 * q + 2] = e.z;
        cin[kEmb + 4 * q + 3] = e.w;
    }
    float c1[kCHidden];
#pragma unroll
    for (int o = 0; o < kCHidden; ++o) {
        float acc = Wc[kCB1 + o];
#pragma unroll
        for (int i = 0; i < kCIn; ++i) acc += Wc[kCW1 + o * kCIn + i] * cin[i];
        c1[o] = acc < 0.f ? 0.f : acc;
    }
    float c2[kCHidden];
#pragma unroll
    for (int o = 0; o < kCHidden; ++o) {
        float acc = Wc[kCB2 + o];
#pragma unroll
        for (int i = 0; i < kCHidden; ++i) acc += Wc[kCW2 + o * kCHidden + i] * c1[i];
        c2[o] = acc < 0.f ? 0.f : acc;
    }
#pragma unroll
    for (int o = 0; o < 3; ++o) {
        float acc = Wc[kCB3 + o];
#pragma unroll
        for (int i = 0; i < kCHidden; ++i) acc += Wc[kCW3 + o * kCHidden + i] * c2[i];
        rgb[o] = sigmoidf_(acc);
    }
}

__global__ void __launch_bounds__(kTile) field_fwd_kernel(FieldArgs a) {
    extern __shared__ float sm[];
    float* Wd = sm;
    float* Wc = sm + kDnetParams;
    const Status* st = a.status;
    uint32_t n_tiles = st->n_tiles;
    load_floats(Wc, a.f.color, kColorParams);
    int cur = -1;
    for (uint32_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
        TileDesc td = a.tiles[t];
        if (td.slot != cur) {
            __syncthreads();
            load_floats(Wd, a.f.dnet[td.slot], kDnetParams);
            cur = td.slot;
            __syncthreads();
        }
        int i = threadIdx.x;
        if (i < td.n) {
            uint64_t pos = uint64_t(td.start) + i;
            float4 L = a.s.local[pos];
            int ray = __float_as_int(L.w);
            float feat[kFeatDim];
            hash_encode(a.hl, a.f.enc[td.slot], L.x, L.y, L.z, feat);
            float sg, rgb[3];
            field_point_fwd(Wd, Wc, feat, a.venc + uint64_t(ray) * 6, a.density_lim,
                            a.density_max, &sg, rgb);
            a.s.io[pos] = make_float4(sg, rgb[0], rgb[1], rgb[2]);
        }
    }
}

void launch_field_forward(const FieldArgs& a, int grid, cudaStream_t st, uint64_t* launches) {
    size_t smem = kFwdSmemFloats * sizeof(float);
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(field_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        attr = true;
    }
    field_fwd_kernel<<<grid, kTile, smem, st>>>(a);
    *launches += 1;
}

// ------------------------------------------------------------------ K4 backward
// Per tile: recompute the forward with every activation of the 128 rows kept
// in shared memory, backpropagate row-locally (data gradients), accumulate
// the weight gradients of the tile as smem GEMMs over its 128 rows into
// block-private accumulators (flushed to global with one atomic per weight
// when the slot changes and at the end), and scatter the hash-table gradient
// with vector atomics (red.global.add.v2.f32).
constexpr int kLdX0 = 17, kLdH1 = 65, kLdO = 17, kLdCin = 41, kLdC1 = 65, kLdC2 = 65, kLdD3 = 4;
constexpr int kActOffX0 = 0;
constexpr int kActOffH1 = kActOffX0 + kTile * kLdX0;
constexpr int kActOffO = kActOffH1 + kTile * kLdH1;
constexpr int kActOffCin = kActOffO + kTile * kLdO;
constexpr int kActOffC1 = kActOffCin + kTile * kLdCin;
constexpr int kActOffC2 = kActOffC1 + kTile * kLdC1;
constexpr int kActOffD3 = kActOffC2 + kTile * kLdC2;
constexpr int kActFloats = kActOffD3 + kTile * kLdD3;
constexpr int kBwdSmemFloats = 2 * kDnetParams + 2 * kColorParams + kActFloats + 2;

// G[o][i] += sum_t D[t][o] * X[t][i] over the 128 rows; gb[o] += sum_t D[t][o].
template <int NO, int NI>
__device__ __forceinline__ void wgrad(const float* D, int ldd, const float* X, int ldx, float* G,
                                      float* gb) {
    for (int e = threadIdx.x; e < NO * NI; e += kTile) {
        int o = e / NI, i = e - o * NI;
        float acc = 0.f;
#pragma unroll 8
        for (int t = 0; t < kTile; ++t) acc += D[t * ldd + o] * X[t * ldx + i];
        G[o * NI + i] += acc;
    }
    for (int o = threadIdx.x; o < NO; o += kTile) {
        float acc = 0.f;
        for (int t = 0; t < kTile; ++t) acc += D[t * ldd + o];
        gb[o] += acc;
    }
}

__device__ __forceinline__ void flush(float* __restrict__ dst, float* src, int n) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        float v = src[i];
        if (v != 0.f) atomicAdd(dst + i, v);
        src[i] = 0.f;
    }
}

__global__ void __launch_bounds__(kTile) field_bwd_kernel(FieldArgs a, FieldGradArgs g) {
    extern __shared__ float sm[];
    float* Wd = sm;
    float* Wc = Wd + kDnetParams;
    float* Gd = Wc + kColorParams;
    float* Gc = Gd + kDnetParams;
    float* act = Gc + kColorParams;
    float* X0 = act + kActOffX0;
    float* H1 = act + kActOffH1;
    float* O = act + kActOffO;
    float* CIN = act + kActOffCin;
    float* C1 = act + kActOffC1;
    float* C2 = act + kActOffC2;
    float* D3 = act + kActOffD3;
    const int r = threadIdx.x;
    uint32_t n_tiles = a.status->n_tiles;
    load_floats(Wc, a.f.color, kColorParams);
    for (int i = threadIdx.x; i < kColorParams; i += blockDim.x) Gc[i] = 0.f;
    for (int i = threadIdx.x; i < kDnetParams; i += blockDim.x) Gd[i] = 0.f;
    int cur = -1;
    for (uint32_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
        TileDesc td = a.tiles[t];
        __syncthreads();
        if (td.slot != cur) {
            if (cur >= 0) flush(g.g_dnet[cur], Gd, kDnetParams);
            load_floats(Wd, a.f.dnet[td.slot], kDnetParams);
            cur = td.slot;
            __syncthreads();
        }
        bool live = r < td.n;
        uint64_t pos = uint64_t(td.start) + r;
        float4 L = make_float4(0.f, 0.f, 0.f, 0.f);
        float4 dio = make_float4(0.f, 0.f, 0.f, 0.f);
        int ray = 0;
        if (live) {
            L = a.s.local[pos];
            ray = __float_as_int(L.w);
            dio = a.s.io[pos];  // (d_sigma, d_r, d_g, d_b) from K3
        }
        // ---- forward recompute into smem rows
        float* x0 = X0 + r * kLdX0;
        float* h1 = H1 + r * kLdH1;
        float* o16 = O + r * kLdO;
        float* cin = CIN + r * kLdCin;
        float* c1 = C1 + r * kLdC1;
        float* c2 = C2 + r * kLdC2;
        float* d3 = D3 + r * kLdD3;
        float feat[kFeatDim];
        if (live) hash_encode(a.hl, a.f.enc[td.slot], L.x, L.y, L.z, feat);
        else
            for (int i = 0; i < kFeatDim; ++i) feat[i] = 0.f;
        for (int i = 0; i < kFeatDim; ++i) x0[i] = feat[i];
        for (int o = 0; o < kDHidden; ++o) {
            float acc = Wd[kDB1 + o];
#pragma unroll
            for (int i = 0; i < kFeatDim; ++i) acc += Wd[kDW1 + o * kFeatDim + i] * feat[i];
            h1[o] = acc < 0.f ? 0.f : acc;
        }
        float draw = 0.f;
        for (int o = 0; o < kDOut; ++o) {
            float acc = Wd[kDB2 + o];
#pragma unroll 16
            for (int i = 0; i < kDHidden; ++i) acc += Wd[kDW2 + o * kDHidden + i] * h1[i];
            if (o == 0) draw = acc >= a.density_lim ? 0.f : expf(acc);
            else cin[o - 1] = acc;
        }
        const float4* ve = a.venc + uint64_t(ray) * 6;
        for (int q = 0; q < 6; ++q) {
            float4 e = live ? __ldg(ve + q) : make_float4(0.f, 0.f, 0.f, 0.f);
            cin[kEmb + 4 * q] = e.x;
            cin[kEmb + 4 * q + 1] = e.y;
            cin[kEmb + 4 * q + 2] = e.z;
            cin[kEmb + 4 * q + 3] = e.w;
        }
        cin[kCIn] = 0.f;
        for (int o = 0; o < kCHidden; ++o) {
            float acc = Wc[kCB1 + o];
#pragma unroll 13
            for (int i = 0; i < kCIn; ++i) acc += Wc[kCW1 + o * kCIn + i] * cin[i];
            c1[o] = acc < 0.f ? 0.f : acc;
        }
        for (int o = 0; o < kCHidden; ++o) {
            float acc = Wc[kCB2 + o];
#pragma unroll 16
            for (int i = 0; i < kCHidden; ++i) acc += Wc[kCW2 + o * kCHidden + i] * c1[i];
            c2[o] = acc < 0.f ? 0.f : acc;
        }
        for (int o = 0; o < 3; ++o) {
            float acc = Wc[kCB3 + o];
#pragma unroll 16
            for (int i = 0; i < kCHidden; ++i) acc += Wc[kCW3 + o * kCHidden + i] * c2[i];
            (void)acc;  // K3 hands over the pre-sigmoid gradient
            float gin = o == 0 ? dio.y : (o == 1 ? dio.z : dio.w);
            d3[o] = live ? gin : 0.f;
        }
        d3[3] = 0.f;
        __syncthreads();
        // ---- colour layer 3: dW3 += d3 (x) c2; then dC2 = W3^T d3 * [c2 > 0] in place
        wgrad<3, kCHidden>(D3, kLdD3, C2, kLdC2, Gc + kCW3, Gc + kCB3);
        __syncthreads();
        for (int i = 0; i < kCHidden; ++i) {
            float acc = 0.f;
#pragma unroll
            for (int o = 0; o < 3; ++o) acc += Wc[kCW3 + o * kCHidden + i] * d3[o];
            c2[i] = c2[i] > 0.f ? acc : 0.f;
        }
        __syncthreads();
        // ---- colour layer 2: dW2 += dC2 (x) c1; dC1 = W2^T dC2 * [c1 > 0] in place
        wgrad<kCHidden, kCHidden>(C2, kLdC2, C1, kLdC1, Gc + kCW2, Gc + kCB2);
        __syncthreads();
        {
            float acc[kCHidden];
#pragma unroll
            for (int i = 0; i < kCHidden; ++i) acc[i] = 0.f;
            for (int o = 0; o < kCHidden; ++o) {
                float d = c2[o];
#pragma unroll
                for (int i = 0; i < kCHidden; ++i) acc[i] += Wc[kCW2 + o * kCHidden + i] * d;
            }
#pragma unroll
            for (int i = 0; i < kCHidden; ++i) c1[i] = c1[i] > 0.f ? acc[i] : 0.f;
        }
        __syncthreads();
        // ---- colour layer 1: dW1 += dC1 (x) cin; d_emb = (W1^T dC1)[0:15]
        wgrad<kCHidden, kCIn>(C1, kLdC1, CIN, kLdCin, Gc + kCW1, Gc + kCB1);
        __syncthreads();
        {
            float acc[kEmb];
#pragma unroll
            for (int i = 0; i < kEmb; ++i) acc[i] = 0.f;
            for (int o = 0; o < kCHidden; ++o) {
                float d = c1[o];
#pragma unroll
                for (int i = 0; i < kEmb; ++i) acc[i] += Wc[kCW1 + o * kCIn + i] * d;
            }
            o16[0] = live ? dio.x : 0.f;  // d raw sigma (K3)
            (void)draw;
#pragma unroll
            for (int i = 0; i < kEmb; ++i) o16[1 + i] = acc[i];
        }
        __syncthreads();
        // ---- density layer 2: dW += dO (x) h1; dH1 = W^T dO * [h1 > 0] in place
        wgrad<kDOut, kDHidden>(O, kLdO, H1, kLdH1, Gd + kDW2, Gd + kDB2);
        __syncthreads();
        {
            float acc[kDHidden];
#pragma unroll
            for (int i = 0; i < kDHidden; ++i) acc[i] = 0.f;
            for (int o = 0; o < kDOut; ++o) {
                float d = o16[o];
#pragma unroll
                for (int i = 0; i < kDHidden; ++i) acc[i] += Wd[kDW2 + o * kDHidden + i] * d;
            }
#pragma unroll
            for (int i = 0; i < kDHidden; ++i) h1[i] = h1[i] > 0.f ? acc[i] : 0.f;
        }
        __syncthreads();
        // ---- density layer 1: dW += dH1 (x) x0; d_feat = W^T dH1 -> hash scatter
        wgrad<kDHidden, kFeatDim>(H1, kLdH1, X0, kLdX0, Gd + kDW1, Gd + kDB1);
        {
            float df[kFeatDim];
#pragma unroll
            for (int i = 0; i < kFeatDim; ++i) df[i] = 0.f;
            for (int o = 0; o < kDHidden; ++o) {
                float d = h1[o];
#pragma unroll
                for (int i = 0; i < kFeatDim; ++i) df[i] += Wd[kDW1 + o * kFeatDim + i] * d;
            }
            if (live) hash_scatter(a.hl, g.g_enc[td.slot], L.x, L.y, L.z, df);
        }
    }
    __syncthreads();
    if (cur >= 0) flush(g.g_dnet[cur], Gd, kDnetParams);
    flush(g.g_color, Gc, kColorParams);
}

void launch_field_backward(const FieldArgs& a, const FieldGradArgs& g, int grid, cudaStream_t st,
                           uint64_t* launches) {
    size_t smem = kBwdSmemFloats * sizeof(float);
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(field_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        attr = true;
    }
    field_bwd_kernel<<<grid, kTile, smem, st>>>(a, g);
    *launches += 1;
}

// ------------------------------------------------------------------ K6 occupancy
// TileField::update_occupancy (field.hpp:100-102): per voxel a
// jittered probe (Rng(hash_combine(base, voxel)): 3 floats), EMA <- max(decay *
// EMA, sigma); bits <- EMA >= threshold.  update == 0 only rebuilds the bits.
__global__ void __launch_bounds__(256) occupancy_kernel(OccArgs a) {
    __shared__ float Wd[kDnetParams];
    int slot = blockIdx.y;
    load_floats(Wd, a.dnet[slot], kDnetParams);
    __syncthreads();
    int v = blockIdx.x * blockDim.x + threadIdx.x;
    float e = a.ema[slot][v];
    if (a.update) {
        int x = v % kOccRes, y = (v / kOccRes) % kOccRes, z = v / (kOccRes * kOccRes);
        Rng rng(hash_combine(a.base_key[slot], uint64_t(v)));
        float ux = rng.flt(), uy = rng.flt(), uz = rng.flt();
        float px = (float(x) + ux) / float(kOccRes);
        float py = (float(y) + uy) / float(kOccRes);
        float pz = (float(z) + uz) / float(kOccRes);
        float feat[kFeatDim];
        hash_encode(a.hl, a.enc[slot], px, py, pz, feat);
        float h[kDHidden];
#pragma unroll
        for (int o = 0; o < kDHidden; ++o) {
            float acc = Wd[kDB1 + o];
#pragma unroll
            for (int i = 0; i < kFeatDim; ++i) acc += Wd[kDW1 + o * kFeatDim + i] * feat[i];
            h[o] = acc < 0.f ? 0.f : acc;
        }
        float raw = Wd[kDB2];
#pragma unroll
        for (int i = 0; i < kDHidden; ++i) raw += Wd[kDW2 + i] * h[i];
        float sg = raw >= a.density_lim ? a.density_max : expf(raw);
        float d = a.decay * e;
        e = d < sg ? sg : d;  // std::max(decay * ema, sigma)
        a.ema[slot][v] = e;
    }
    uint32_t bit = e >= a.threshold ? 1u : 0u;
    uint32_t word = __ballot_sync(0xffffffffu, bit);
    if ((threadIdx.x & 31) == 0) a.bits[slot][v >> 5] = word;
}

void launch_occupancy(const OccArgs& a, cudaStream_t st, uint64_t* launches) {
    dim3 grid(kOccVox / 256, a.n);
    occupancy_kernel<<<grid, 256, 0, st>>>(a);
    *launches += 1;
}

} // namespace tfg
