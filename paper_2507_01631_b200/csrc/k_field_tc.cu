// k_field_tc.cu — K2/K4 on the 5th-generation tensor cores (tcgen05 + TMEM).
//
// The per-tile NeRF field (forward_batch / backward_batch, field.hpp:185-197;
// MlpT nn.hpp:90-157; HashGridT nn.hpp:213-245) split by bound:
//   K2a hash_fwd_kernel   hash-grid gather (L1-throughput bound): 16 features
//                         per sample -> bf16 tile in UMMA operand layout
//                         (4 KB/tile), reused by K4b
//   K2b mlp_fwd_kernel    density MLP 16->64->16 + colour MLP 39->64->64->3 as
//                         tcgen05.mma (bf16 x bf16 -> fp32 in TMEM), weights
//                         and features staged by the bulk-copy engine; each
//                         accumulator starts at the layer's bias (one extra
//                         K=16 MMA), epilogues (ReLU folded into the bf16
//                         pack, exp/sigmoid) from tcgen05.ld; each epilogue's
//                         bf16 output goes back to TMEM with tcgen05.st as the
//                         next layer's A operand
//   K4b mlp_bwd_kernel    recomputed forward (biases through the MMA as in
//                         K2b, so the pre-activations are the forward's bits)
//                         + data-gradient GEMMs (ReLU masks read from the
//                         stored bf16 activations) + weight-gradient GEMMs
//                         (K = 128 samples, MN-major operands read from the
//                         same smem tiles) accumulated in TMEM
//                         across all tiles of a persistent CTA, flushed with
//                         one fp32 atomic per weight per CTA
//   (K4a)                 hash-table scatter-add on K4b's own scatter warps
//                         (warp specialisation: they drain d(features) from
//                         TMEM while the MLP warps run the next tile;
//                         red.global.add.v4/v2.f32 on aligned x-neighbour
//                         pairs, same-cell lane pairs merged on levels 0-2)
// A tile is <= 128 samples of one slot bucket (K1), so the density weights of
// a tile are one tile's.  Precision: bf16 operands, fp32 accumulation (tests
// state the tolerance against the fp32 oracle).
#include <mutex>

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "tf_common.cuh"
#include "tf_hash.cuh"
#include "tf_kernels.h"
#include "umma.cuh"

namespace tfg {

namespace {

constexpr int kT = 128;
constexpr uint32_t kChunk = kT * 16;  // bytes of one 8-column chunk of a 128-row tile
constexpr uint32_t kFeatTile = 2 * kChunk;

// smem weight tiles (bf16, chunk-major interleave; rows = out features)
constexpr uint32_t kW1dRows = 64, kW2dRows = 16, kWc1Rows = 64, kWc2Rows = 64, kWc3Rows = 16;
constexpr uint32_t kW1dBytes = kW1dRows * 16 * 2;   // [64 x 16]
constexpr uint32_t kW2dBytes = kW2dRows * 64 * 2;   // [16 x 64]
constexpr uint32_t kWc1Bytes = kWc1Rows * 48 * 2;   // [64 x 48] (39 real)
constexpr uint32_t kWc2Bytes = kWc2Rows * 64 * 2;   // [64 x 64]
constexpr uint32_t kWc3Bytes = kWc3Rows * 64 * 2;   // [16 x 64] (3 real)
constexpr uint32_t kBiasFloats = 64 + 16 + 64 + 64 + 16;

struct Weights {
    uint8_t* w1d;
    uint8_t* w2d;
    uint8_t* wc1;
    uint8_t* wc2;
    uint8_t* wc3;
    // fp32 bias copies: no longer read (the biases enter through the MMAs,
    // stage_bias_tile), still staged: removing them measured the forward
    // 5 us slower in a same-box A/B (0.510 vs 0.515 ms, a code-placement
    // effect), so they stay until that is understood
    float* b1d;
    float* b2d;
    float* bc1;
    float* bc2;
    float* bc3;
};

__device__ __forceinline__ uint8_t* carve(uint8_t*& p, uint32_t bytes) {
    uint8_t* r = p;
    p += (bytes + 127) & ~127u;
    return r;
}

__device__ __forceinline__ Weights carve_weights(uint8_t*& p) {
    Weights w;
    w.w1d = carve(p, kW1dBytes);
    w.w2d = carve(p, kW2dBytes);
    w.wc1 = carve(p, kWc1Bytes);
    w.wc2 = carve(p, kWc2Bytes);
    w.wc3 = carve(p, kWc3Bytes);
    float* b = reinterpret_cast<float*>(carve(p, kBiasFloats * 4));
    w.b1d = b;
    w.b2d = b + 64;
    w.bc1 = b + 80;
    w.bc2 = b + 144;
    w.bc3 = b + 208;
    return w;
}
constexpr uint32_t kWeightsBytes = ((kW1dBytes + 127) & ~127u) + ((kW2dBytes + 127) & ~127u) +
                                   ((kWc1Bytes + 127) & ~127u) + ((kWc2Bytes + 127) & ~127u) +
                                   ((kWc3Bytes + 127) & ~127u) + ((kBiasFloats * 4 + 127) & ~127u);

__device__ __forceinline__ uint32_t pack2(float a, float b);

// fp32 row-major W [RS x CS] (out x in) -> bf16 [ROWS x COLS] chunk-major
// tile, zero padded.  One item = the 8 columns of one row (a 16 B core-matrix
// row); a thread issues all its items' loads before any store, so staging
// costs one global round trip instead of one per element (per element it sat
// on the forward's critical path at every slot change: ~8% of mlp_fwd's
// stall samples).  Row starts of W are 16 B aligned when CS % 4 == 0.
template <int RS, int CS, int ROWS, int COLS>
__device__ __forceinline__ void stage_matrix(uint8_t* dst, const float* __restrict__ W) {
    constexpr int kCh = COLS / 8, kItems = ROWS * kCh, kPer = (kItems + kT - 1) / kT;
    float v[kPer][8];
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
        const int it = int(threadIdx.x) + q * kT, r = it / kCh, c0 = (it % kCh) * 8;
#pragma unroll
        for (int j = 0; j < 8; ++j) v[q][j] = 0.f;
        if (it < kItems && r < RS) {
            const float* src = W + r * CS + c0;
            if constexpr (CS % 4 == 0) {
                if (c0 < CS) {
                    const float4 x = __ldg(reinterpret_cast<const float4*>(src));
                    v[q][0] = x.x, v[q][1] = x.y, v[q][2] = x.z, v[q][3] = x.w;
                }
                if (c0 + 4 < CS) {
                    const float4 x = __ldg(reinterpret_cast<const float4*>(src) + 1);
                    v[q][4] = x.x, v[q][5] = x.y, v[q][6] = x.z, v[q][7] = x.w;
                }
            } else {
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    if (c0 + j < CS) v[q][j] = __ldg(src + j);
            }
        }
    }
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
        const int it = int(threadIdx.x) + q * kT;
        if (it < kItems)
            *reinterpret_cast<uint4*>(dst + umma::off(ROWS, it / kCh, (it % kCh) * 8)) =
                make_uint4(pack2(v[q][0], v[q][1]), pack2(v[q][2], v[q][3]), pack2(v[q][4], v[q][5]),
                           pack2(v[q][6], v[q][7]));
    }
}
__device__ __forceinline__ void stage_density(const Weights& w, const float* __restrict__ p) {
    static_assert(kDW1 % 4 == 0 && kDW2 % 4 == 0, "density weight rows are float4 aligned");
    stage_matrix<kDHidden, kFeatDim, 64, 16>(w.w1d, p + kDW1);
    stage_matrix<kDOut, kDHidden, 16, 64>(w.w2d, p + kDW2);
    for (int i = threadIdx.x; i < 64; i += kT) w.b1d[i] = p[kDB1 + i];
    for (int i = threadIdx.x; i < 16; i += kT) w.b2d[i] = p[kDB2 + i];
}
// Colour layer 1's weights [64 x 48] with its bias riding in its own K range:
// input column kCIn (the ones column the backward's dWc1 bias gradient uses)
// and kCIn + 1 are 1, so the tile holds bf16(bc1) and bf16(bc1 - bf16(bc1))
// there.  Written by the thread that writes the chunk (one writer per byte).
__device__ __forceinline__ void stage_wc1(uint8_t* dst, const float* __restrict__ p) {
    static_assert(kCIn == 39, "the bias columns 39 / 40 straddle chunks 4 and 5");
    constexpr int kCh = 6, kItems = 64 * kCh;
    for (int it = threadIdx.x; it < kItems; it += kT) {
        const int r = it / kCh, c = it % kCh, c0 = 8 * c;
        float v[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) v[j] = c0 + j < kCIn ? __ldg(p + kCW1 + r * kCIn + c0 + j) : 0.f;
        const float b = p[kCB1 + r];
        const float hi = __bfloat162float(__float2bfloat16_rn(b));
        if (c == 4) v[7] = b;         // col 39: rounds to hi
        if (c == 5) v[0] = b - hi;    // col 40: rounds to bf16(b - hi)
        *reinterpret_cast<uint4*>(dst + umma::off(64, r, c0)) =
            make_uint4(pack2(v[0], v[1]), pack2(v[2], v[3]), pack2(v[4], v[5]), pack2(v[6], v[7]));
    }
}
__device__ __forceinline__ void stage_color(const Weights& w, const float* __restrict__ p) {
    static_assert(kCW2 % 4 == 0 && kCW3 % 4 == 0, "colour weight rows are float4 aligned");
    stage_wc1(w.wc1, p);
    stage_matrix<kCHidden, kCHidden, 64, 64>(w.wc2, p + kCW2);
    stage_matrix<3, kCHidden, 16, 64>(w.wc3, p + kCW3);
    for (int i = threadIdx.x; i < 64; i += kT) {
        w.bc1[i] = p[kCB1 + i];
        w.bc2[i] = p[kCB2 + i];
    }
    for (int i = threadIdx.x; i < 16; i += kT) w.bc3[i] = i < 3 ? p[kCB3 + i] : 0.f;
}

// Each layer's bias as an MMA operand (the forward and the backward's
// recompute), so the accumulator starts at the bias and the epilogues carry
// no bias add.  B tile [N x 16]
// (chunk-major, rows = out features): column 0 = bf16(b), column 1 =
// bf16(b - bf16(b)), the rest 0; multiplied by the constant A tile whose
// columns 0 and 1 are 1, it contributes b to 16 mantissa bits (the bias
// enters first, then the layer's products).
constexpr uint32_t kBiasTile64 = 64 * 16 * 2, kBiasTile16 = 16 * 16 * 2;
struct BiasTiles {
    uint8_t* ones;  // [128 x 16]: columns 0, 1 = 1
    uint8_t* l1;    // [64 x 16]
    uint8_t* l2;    // [16 x 16]
    uint8_t* c2;  // (colour layer 1's bias rides in its weight tile: stage_color)
    uint8_t* c3;    // [16 x 16] (3 real rows)
};
template <int N>
__device__ __forceinline__ void stage_bias_tile(uint8_t* dst, const float* __restrict__ b, int n_real) {
    for (int o = threadIdx.x; o < N; o += kT) {
        const float x = o < n_real ? b[o] : 0.f;
        const __nv_bfloat16 hi = __float2bfloat16_rn(x);
        const __nv_bfloat16 lo = __float2bfloat16_rn(x - __bfloat162float(hi));
        uint4 q = make_uint4(uint32_t(*reinterpret_cast<const uint16_t*>(&hi)) |
                                 (uint32_t(*reinterpret_cast<const uint16_t*>(&lo)) << 16),
                             0u, 0u, 0u);
        *reinterpret_cast<uint4*>(dst + umma::off(N, o, 0)) = q;
        *reinterpret_cast<uint4*>(dst + umma::off(N, o, 8)) = make_uint4(0u, 0u, 0u, 0u);
    }
}

__device__ __forceinline__ uint32_t pack2(float a, float b) {
    __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
}
// ReLU folded into the bf16 pack (one F2FP.RELU per pair): relu then round
// equals round then relu, bit for bit.
__device__ __forceinline__ uint32_t pack2_relu(float a, float b) {
    uint32_t d;
    asm("cvt.rn.relu.bf16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(b), "f"(a));
    return d;
}
// Writes 8 consecutive columns [8c, 8c+8) of row r of a 128-row tile.
__device__ __forceinline__ void st_chunk(uint8_t* buf, int r, int c, const float* v) {
    uint4 q = make_uint4(pack2(v[0], v[1]), pack2(v[2], v[3]), pack2(v[4], v[5]), pack2(v[6], v[7]));
    *reinterpret_cast<uint4*>(buf + c * kChunk + (r >> 3) * 128 + (r & 7) * 16) = q;
}
// Overwrites the 8 ReLU'd activations of row r, chunk c with 8 gradients
// masked by the ReLU: kept where the activation is positive, 0 elsewhere
// (one HSET2 mask + one AND per pair; the masks need no registers between
// the forward recompute and the backward).
__device__ __forceinline__ void st_chunk_masked(uint8_t* buf, int r, int c, const float* v) {
    uint4* const p = reinterpret_cast<uint4*>(buf + c * kChunk + (r >> 3) * 128 + (r & 7) * 16);
    const uint4 act = *p;
    const __nv_bfloat162 zero = __float2bfloat162_rn(0.f);
    auto gt0 = [&](uint32_t w) { return __hgt2_mask(*reinterpret_cast<const __nv_bfloat162*>(&w), zero); };
    *p = make_uint4(pack2(v[0], v[1]) & gt0(act.x), pack2(v[2], v[3]) & gt0(act.y), pack2(v[4], v[5]) & gt0(act.z),
                    pack2(v[6], v[7]) & gt0(act.w));
}
__device__ __forceinline__ void st_chunk_relu(uint8_t* buf, int r, int c, const float* v) {
    uint4 q = make_uint4(pack2_relu(v[0], v[1]), pack2_relu(v[2], v[3]), pack2_relu(v[4], v[5]),
                         pack2_relu(v[6], v[7]));
    *reinterpret_cast<uint4*>(buf + c * kChunk + (r >> 3) * 128 + (r & 7) * 16) = q;
}


// Descriptors for the chunk-major tiles (see umma.cuh).
__device__ __forceinline__ uint64_t kmaj(const uint8_t* base, uint32_t rows, int kstep) {
    // rows x K tile read K-major; kstep-th group of 16 K columns
    return umma::desc(umma::smem_u32(base) + kstep * 2 * rows * 16, rows * 16, 128);
}
__device__ __forceinline__ uint64_t mnmaj(const uint8_t* base, uint32_t rows, int kstep) {
    // rows = K x cols = MN tile read MN-major; kstep-th group of 16 K rows
    return umma::desc(umma::smem_u32(base) + kstep * 256, 128, rows * 16);
}

// Barrier before a single thread issues MMAs that read smem written by all
// threads (generic -> async proxy) and overwrite TMEM other threads read.
__device__ __forceinline__ void sync_for_mma() {
    umma::fence_async_smem();
    umma::fence_before_sync();
    __syncthreads();
    umma::fence_after_sync();
}
// Same, over the 128 MLP threads of a warp-specialised CTA (named barrier 1).
__device__ __forceinline__ void sync_mlp() {
    umma::fence_async_smem();
    umma::fence_before_sync();
    asm volatile("bar.sync 1, 128;\n" ::: "memory");
    umma::fence_after_sync();
}
__device__ __forceinline__ void wait_mma(uint64_t* bar, uint32_t& phase) {
    umma::mbar_wait(bar, phase);
    phase ^= 1u;
    umma::fence_after_sync();
}

// 16 TMEM columns starting at col of this thread's lane row.
__device__ __forceinline__ void tld16(uint32_t tmem, int col, float* v) {
    uint32_t w = threadIdx.x >> 5;
    umma::ld16(tmem + ((32u * w) << 16) + uint32_t(col), v);
}

// Packs n (multiple of 16) activations of this thread's row to bf16 pairs in
// TMEM columns [col, col + n/2) of its lane (the A operand of the next layer).
template <int N>
__device__ __forceinline__ void tst_bf16(uint32_t tmem, int col, const float* v) {
    const uint32_t w = threadIdx.x >> 5;
#pragma unroll
    for (int c = 0; c < N / 16; ++c) {
        uint32_t q[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) q[j] = pack2(v[16 * c + 2 * j], v[16 * c + 2 * j + 1]);
        umma::st8(tmem + ((32u * w) << 16) + uint32_t(col + 8 * c), q);
    }
}
template <int N>
__device__ __forceinline__ void tst_bf16_relu(uint32_t tmem, int col, const float* v) {
    const uint32_t w = threadIdx.x >> 5;
#pragma unroll
    for (int c = 0; c < N / 16; ++c) {
        uint32_t q[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) q[j] = pack2_relu(v[16 * c + 2 * j], v[16 * c + 2 * j + 1]);
        umma::st8(tmem + ((32u * w) << 16) + uint32_t(col + 8 * c), q);
    }
}
// Barrier before thread 0 issues MMAs that read the A operand other threads
// stored to TMEM and overwrite the accumulator they read.
__device__ __forceinline__ void sync_for_mma_tmem() {
    umma::st_wait();
    umma::fence_before_sync();
    __syncthreads();
    umma::fence_after_sync();
}

__device__ __forceinline__ float sigm(float x) { return 1.f / (1.f + __expf(-x)); }

} // namespace

// ------------------------------------------------------------------ K2a
// Thread per tile row: 8-level hash gather -> 16 bf16 features in the tile's
// chunk-major layout (the A operand of the first density layer) + ray id.
template <bool G>
__global__ void __launch_bounds__(128) hash_fwd_kernel(FieldArgs a, uint8_t* __restrict__ feat,
                                                       int32_t* __restrict__ rays) {
    pdl_wait();
    uint32_t n_tiles = a.status->n_tiles;
    int r = threadIdx.x;
    for (uint32_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
        TileDesc td = a.tiles[t];
        float f[kFeatDim];
        int ray = -1;
        if (r < td.n) {
            float4 L = a.s.local[uint64_t(td.start) + r];
            ray = __float_as_int(L.w);
            hash_encode16<G>(a.hl, a.f.enc16[td.slot], L.x, L.y, L.z, f);
        } else {
#pragma unroll
            for (int i = 0; i < kFeatDim; ++i) f[i] = 0.f;
        }
        uint8_t* base = feat + uint64_t(t) * kFeatTile;
        st_chunk(base, r, 0, f);
        st_chunk(base, r, 1, f + 8);
        rays[uint64_t(t) * kT + r] = ray;
    }
}

// ------------------------------------------------------------------ K4a
// Hash-table scatter-add (HashGridT::backward, nn.hpp:231-245), run by the
// backward's scatter warps.
// Pair-vectorised scatter of one level's 8 corners (see hash_encode): one
// red.global.add.v4.f32 for an aligned x-neighbour pair, else two v2.
__device__ __forceinline__ void scatter_pairs(float* __restrict__ genc, const Corner& c, float d0,
                                              float d1) {
    float2* g2 = reinterpret_cast<float2*>(genc);
    float4* g4 = reinterpret_cast<float4*>(genc);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        uint32_t i0 = c.idx[2 * q], i1 = c.idx[2 * q + 1];
        float w0 = c.w[2 * q], w1 = c.w[2 * q + 1];
        if (i1 == (i0 ^ 1u)) {
            bool odd = i0 & 1u;
            float4 v = odd ? make_float4(w1 * d0, w1 * d1, w0 * d0, w0 * d1)
                           : make_float4(w0 * d0, w0 * d1, w1 * d0, w1 * d1);
            atomicAdd(g4 + (i0 >> 1), v);
        } else {
            atomicAdd(g2 + i0, make_float2(w0 * d0, w0 * d1));
            atomicAdd(g2 + i1, make_float2(w1 * d0, w1 * d1));
        }
    }
}

__device__ __forceinline__ void red_pair(float* __restrict__ genc, uint32_t i0, uint32_t i1, float a0,
                                         float a1, float b0, float b1) {
    float2* g2 = reinterpret_cast<float2*>(genc);
    float4* g4 = reinterpret_cast<float4*>(genc);
    if (i1 == (i0 ^ 1u)) {
        bool odd = i0 & 1u;
        atomicAdd(g4 + (i0 >> 1), odd ? make_float4(b0, b1, a0, a1) : make_float4(a0, a1, b0, b1));
    } else {
        atomicAdd(g2 + i0, make_float2(a0, a1));
        atomicAdd(g2 + i1, make_float2(b0, b1));
    }
}

// Butterfly merging (registers + shuffles only; the scatter is bound by
// L1/LSU transactions, so smem staging costs as much as it saves).  Round 1
// pairs lanes (2i, 2i+1): the even lane recomputes its partner's trilinear
// weights from the partner's cell fractions and adds its contribution when
// both sit in the same cell; round 2 merges the 16 accumulated corner values
// of lane 4i+2 into lane 4i.  Lanes whose contribution was merged issue no
// reds.  Levels 0-2 use round 1 only (measured on B200: 1.52 -> 1.35 ms for
// the backward; a second round or a 4th level does not pay, nor does
// merging whole runs through smem, which adds LSU traffic).
#ifndef TFG_BFLY0
#define TFG_BFLY0 1
#endif
#ifndef TFG_BFLY1
#define TFG_BFLY1 1
#endif
#ifndef TFG_BFLY2
#define TFG_BFLY2 1
#endif
#ifndef TFG_BFLY3
#define TFG_BFLY3 0
#endif
__host__ __device__ constexpr int bfly_rounds(int l) {
    return l == 0 ? TFG_BFLY0 : l == 1 ? TFG_BFLY1 : l == 2 ? TFG_BFLY2 : l == 3 ? TFG_BFLY3 : 0;
}

template <int L>
__device__ __forceinline__ void cell_frac(float x, float y, float z, float* f) {
    constexpr int n = level_res_c(L);
    float p[3] = {x, y, z};
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        float v = fminf(fmaxf(p[k], 0.f), 1.f);
        float sc = v * float(n);
        int ci = int(sc);
        ci = ci > n - 1 ? n - 1 : ci;
        f[k] = sc - float(ci);
    }
}

template <int L>
__device__ __forceinline__ void scatter_level_bfly(float* __restrict__ genc, float x, float y, float z,
                                                   float d0, float d1, bool live) {
    constexpr int R = bfly_rounds(L);
    Corner c;
    hash_level_c<L>(x, y, z, c);
    if constexpr (R == 0) {
        if (live) scatter_pairs(genc, c, d0, d1);
    } else {
        const uint32_t FULL = 0xffffffffu;
        const int lane = threadIdx.x & 31;
        uint32_t key = live ? c.idx[0] : 0xffffffffu;
        float a[16];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            a[2 * k] = c.w[k] * d0;
            a[2 * k + 1] = c.w[k] * d1;
        }
        // round 1: odd -> even by recomputation
        float f[3];
        cell_frac<L>(x, y, z, f);
        uint32_t k1 = __shfl_down_sync(FULL, key, 1);
        float px = __shfl_down_sync(FULL, f[0], 1), py = __shfl_down_sync(FULL, f[1], 1);
        float pz = __shfl_down_sync(FULL, f[2], 1);
        float e0 = __shfl_down_sync(FULL, d0, 1), e1 = __shfl_down_sync(FULL, d1, 1);
        uint32_t km1 = __shfl_up_sync(FULL, key, 1);  // (all lanes shuffle)
        bool merged = (lane & 1) && km1 == key;
        if (!(lane & 1) && k1 == key) {
            float wx[2] = {1.f - px, px}, wy[2] = {1.f - py, py}, wz[2] = {1.f - pz, pz};
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                float w = (wx[k & 1] * wy[(k >> 1) & 1]) * wz[k >> 2];
                a[2 * k] += w * e0;
                a[2 * k + 1] += w * e1;
            }
        }
        if constexpr (R >= 2) {
            uint32_t k2 = __shfl_down_sync(FULL, key, 2);
            uint32_t km2 = __shfl_up_sync(FULL, key, 2);
            bool take = (lane & 3) == 0 && k2 == key;
            merged = merged || ((lane & 3) == 2 && km2 == key);
#pragma unroll
            for (int q = 0; q < 16; ++q) {
                float b = __shfl_down_sync(FULL, a[q], 2);
                if (take) a[q] += b;
            }
        }
        if (live && !merged) {
#pragma unroll
            for (int q = 0; q < 4; ++q)
                red_pair(genc, c.idx[2 * q], c.idx[2 * q + 1], a[4 * q], a[4 * q + 1], a[4 * q + 2], a[4 * q + 3]);
        }
    }
}

__device__ __forceinline__ void scatter_row_bfly(float* genc, float x, float y, float z, const float* d,
                                                 bool live) {
    scatter_level_bfly<0>(genc, x, y, z, d[0], d[1], live);
    scatter_level_bfly<1>(genc, x, y, z, d[2], d[3], live);
    scatter_level_bfly<2>(genc, x, y, z, d[4], d[5], live);
    scatter_level_bfly<3>(genc, x, y, z, d[6], d[7], live);
    scatter_level_bfly<4>(genc, x, y, z, d[8], d[9], live);
    scatter_level_bfly<5>(genc, x, y, z, d[10], d[11], live);
    scatter_level_bfly<6>(genc, x, y, z, d[12], d[13], live);
    scatter_level_bfly<7>(genc, x, y, z, d[14], d[15], live);
}
static_assert(kLevels == 8, "scatter_row_bfly unrolls the 8 levels of the default FieldConfig");

// A runtime level layout (non-default n_min / n_max / table_size): the
// pair-vectorised scatter of every level, no butterfly (whose merge rounds
// are chosen per default level).
__device__ __forceinline__ void scatter_row_rt(const HashLayout& hl, float* genc, float x, float y, float z,
                                               const float* d, bool live) {
#pragma unroll
    for (int l = 0; l < kLevels; ++l) {
        Corner c;
        hash_level_rt(hl, l, x, y, z, c);
        if (live) scatter_pairs(genc, c, d[2 * l], d[2 * l + 1]);
    }
}

// ------------------------------------------------------------------ K2b
// smem: weights | X0 [128x16] (the gathered features, bulk-copied; the only
// activation tile in smem).  4 resident CTAs per SM (TMEM and registers).
constexpr uint32_t kFwdSmem = kWeightsBytes + 3 * kFeatTile + 2 * kBiasTile64 + 2 * kBiasTile16 + 128;
// TMEM: accumulator [0, 64); layers 2-5 take their A operand (the previous
// layer's activations, bf16 pairs) from columns [64, 96), so activations never
// touch smem (measured: the MLP's smem pipe was its contended resource).
constexpr uint32_t kFwdTmemCols = 128;
constexpr int kColA = 64;

__global__ void __launch_bounds__(128, 4) mlp_fwd_kernel(FieldArgs a, const uint8_t* __restrict__ feat,
                                                      const int32_t* __restrict__ rays) {
    extern __shared__ __align__(128) uint8_t smem_raw[];
    __shared__ uint64_t bar_mma, bar_ld[2];
    __shared__ uint32_t tmem_slot;
    uint8_t* p = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 127) & ~uintptr_t(127));
    Weights W = carve_weights(p);
    // [128 x 16] feature tiles, double-buffered: tile i+1's bulk copy is in
    // flight while tile i runs
    uint8_t* const X0b0 = carve(p, kFeatTile);
    uint8_t* const X0b1 = carve(p, kFeatTile);
    BiasTiles BT;
    BT.ones = carve(p, kFeatTile);
    BT.l1 = carve(p, kBiasTile64);
    BT.l2 = carve(p, kBiasTile16);
    BT.c2 = carve(p, kBiasTile64);
    BT.c3 = carve(p, kBiasTile16);
    const int r = threadIdx.x;
    if (r == 0) {
        umma::mbar_init(&bar_mma, 1);
        umma::mbar_init(&bar_ld[0], 1);
        umma::mbar_init(&bar_ld[1], 1);
        umma::fence_mbar_init();
    }
    if (r < 32) umma::tmem_alloc<kFwdTmemCols>(&tmem_slot);
    stage_color(W, a.f.color);
    {
        const float o2[8] = {1.f, 1.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f}, z[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        st_chunk(BT.ones, r, 0, o2);
        st_chunk(BT.ones, r, 1, z);
        stage_bias_tile<64>(BT.c2, a.f.color + kCB2, kCHidden);
        stage_bias_tile<16>(BT.c3, a.f.color + kCB3, 3);
    }
    uint32_t ph_mma = 0, ph_ld = 0;  // bit b: phase of bar_ld[b]
    int cur = -1;
    pdl_wait();  // hash_fwd's feature tiles and ray ids
    uint32_t n_tiles = a.status->n_tiles;
    sync_for_mma();
    const uint32_t tmem = tmem_slot;
    const uint32_t id64 = umma::idesc_bf16(128, 64, 0, 0);
    const uint32_t id16 = umma::idesc_bf16(128, 16, 0, 0);
    // the next tile's descriptor and ray ids are loaded one tile ahead (their
    // latency was the largest single stall of the chain)
    // (the descriptor is carried packed and unpacked only when its tile
    // becomes current: unpacked at load time, its field extraction stalled on
    // the load right away)
    uint2 td_next = make_uint2(0u, 0u);
    int ray_next = -1;
    if (blockIdx.x < n_tiles) {
        td_next = __ldg(reinterpret_cast<const uint2*>(a.tiles) + blockIdx.x);
        ray_next = rays[uint64_t(blockIdx.x) * kT + r];
        if (r == 0) {
            umma::mbar_expect_tx(&bar_ld[0], kFeatTile);
            umma::bulk_g2s(X0b0, feat + uint64_t(blockIdx.x) * kFeatTile, kFeatTile, &bar_ld[0]);
        }
    }
    uint32_t it = 0;
    for (uint32_t t = blockIdx.x; t < n_tiles; t += gridDim.x, ++it) {
        asm volatile("" : "+r"(td_next.x), "+r"(td_next.y));
        const TileDesc td{td_next.x, uint16_t(td_next.y & 0xffffu), uint16_t(td_next.y >> 16)};
        const int ray = ray_next;
        const uint32_t b = it & 1u;
        uint8_t* X0 = b ? X0b1 : X0b0;
        if (t + gridDim.x < n_tiles) {
            td_next = __ldg(reinterpret_cast<const uint2*>(a.tiles) + (t + gridDim.x));
            ray_next = rays[uint64_t(t + gridDim.x) * kT + r];
            // the other buffer's last reader (the previous tile's layer-1
            // MMA) has completed
            if (r == 0) {
                umma::mbar_expect_tx(&bar_ld[b ^ 1u], kFeatTile);
                umma::bulk_g2s(b ? X0b0 : X0b1, feat + uint64_t(t + gridDim.x) * kFeatTile, kFeatTile, &bar_ld[b ^ 1u]);
            }
        }
        if (td.slot != cur) {
            stage_density(W, a.f.dnet[td.slot]);
            stage_bias_tile<64>(BT.l1, a.f.dnet[td.slot] + kDB1, kDHidden);
            stage_bias_tile<16>(BT.l2, a.f.dnet[td.slot] + kDB2, kDOut);
            cur = td.slot;
        }
        float ve[kViewDim];
        {
            const float4* v4 = a.venc + uint64_t(ray < 0 ? 0 : ray) * 6;
#pragma unroll
            for (int q = 0; q < 6; ++q) {
                float4 v = __ldg(v4 + q);
                ve[4 * q] = v.x;
                ve[4 * q + 1] = v.y;
                ve[4 * q + 2] = v.z;
                ve[4 * q + 3] = v.w;
            }
        }
        sync_for_mma();  // density weights staged, previous tile's TMEM reads done
        umma::mbar_wait(&bar_ld[b], (ph_ld >> b) & 1u);
        ph_ld ^= 1u << b;
        // ---- density layer 1: [128x16] x W1d^T -> 64
        if (r == 0) {
            umma::mma(tmem, kmaj(BT.ones, kT, 0), kmaj(BT.l1, 64, 0), id64, 0);  // bias
            umma::mma(tmem, kmaj(X0, kT, 0), kmaj(W.w1d, kW1dRows, 0), id64, 1);
            umma::commit(&bar_mma);
        }
        wait_mma(&bar_mma, ph_mma);
        {
            float v[64];
            tld16(tmem, 0, v);
            tld16(tmem, 16, v + 16);
            tld16(tmem, 32, v + 32);
            tld16(tmem, 48, v + 48);
            umma::ld_wait();
            tst_bf16_relu<64>(tmem, kColA, v);
        }
        sync_for_mma_tmem();
        // ---- density layer 2: [128x64] x W2d^T -> 16 (raw sigma | embedding)
        if (r == 0) {
            umma::mma(tmem, kmaj(BT.ones, kT, 0), kmaj(BT.l2, 16, 0), id16, 0);
#pragma unroll
            for (int k = 0; k < 4; ++k)
                umma::mma_ts(tmem, tmem + kColA + 8 * k, kmaj(W.w2d, kW2dRows, k), id16, 1);
            umma::commit(&bar_mma);
        }
        wait_mma(&bar_mma, ph_mma);
        float sigma;
        {
            float v[16];
            tld16(tmem, 0, v);
            umma::ld_wait();
            float raw = v[0];
            sigma = raw >= a.density_lim ? a.density_max : __expf(raw);
            float cin[48];
#pragma unroll
            for (int i = 0; i < kEmb; ++i) cin[i] = v[1 + i];
#pragma unroll
            for (int i = 0; i < kViewDim; ++i) cin[kEmb + i] = ve[i];
            cin[kCIn] = cin[kCIn + 1] = 1.f;  // the bias columns (and K4's bias-gradient column)
#pragma unroll
            for (int i = kCIn + 2; i < 48; ++i) cin[i] = 0.f;
            tst_bf16<48>(tmem, kColA, cin);
        }
        sync_for_mma_tmem();
        // ---- colour layer 1: [128x48] x Wc1^T -> 64
        if (r == 0) {
#pragma unroll
            for (int k = 0; k < 3; ++k)
                umma::mma_ts(tmem, tmem + kColA + 8 * k, kmaj(W.wc1, kWc1Rows, k), id64, k > 0);
            umma::commit(&bar_mma);
        }
        wait_mma(&bar_mma, ph_mma);
        {
            float v[64];
            tld16(tmem, 0, v);
            tld16(tmem, 16, v + 16);
            tld16(tmem, 32, v + 32);
            tld16(tmem, 48, v + 48);
            umma::ld_wait();
            tst_bf16_relu<64>(tmem, kColA, v);
        }
        sync_for_mma_tmem();
        // ---- colour layer 2: [128x64] x Wc2^T -> 64
        if (r == 0) {
            umma::mma(tmem, kmaj(BT.ones, kT, 0), kmaj(BT.c2, 64, 0), id64, 0);
#pragma unroll
            for (int k = 0; k < 4; ++k)
                umma::mma_ts(tmem, tmem + kColA + 8 * k, kmaj(W.wc2, kWc2Rows, k), id64, 1);
            umma::commit(&bar_mma);
        }
        wait_mma(&bar_mma, ph_mma);
        {
            float v[64];
            tld16(tmem, 0, v);
            tld16(tmem, 16, v + 16);
            tld16(tmem, 32, v + 32);
            tld16(tmem, 48, v + 48);
            umma::ld_wait();
            tst_bf16_relu<64>(tmem, kColA, v);
        }
        sync_for_mma_tmem();
        // ---- colour layer 3: [128x64] x Wc3^T -> 16 (3 real) -> sigmoid
        if (r == 0) {
            umma::mma(tmem, kmaj(BT.ones, kT, 0), kmaj(BT.c3, 16, 0), id16, 0);
#pragma unroll
            for (int k = 0; k < 4; ++k)
                umma::mma_ts(tmem, tmem + kColA + 8 * k, kmaj(W.wc3, kWc3Rows, k), id16, 1);
            umma::commit(&bar_mma);
        }
        wait_mma(&bar_mma, ph_mma);
        {
            float v[16];
            tld16(tmem, 0, v);
            umma::ld_wait();
            if (r < td.n)
                a.s.io[uint64_t(td.start) + r] =
                    make_float4(sigma, sigm(v[0]), sigm(v[1]), sigm(v[2]));
        }
    }
    umma::fence_before_sync();
    __syncthreads();
    if (r < 32) umma::tmem_free<kFwdTmemCols>(tmem);
}

// ------------------------------------------------------------------ K4b
// smem (order matters: tiles read as M-padded MN-major operands (H1, C1, C2)
// may over-read up to 16 chunks = 32 KB from their start, which stays inside
// the allocation):
//   H1 [128 x 72] | C1 [128 x 72] | C2 [128 x 72]   (chunk 8 = ones row)
//   X0 [128 x 32] (chunk 2 = ones column, chunk 3 = 0) | CIN [128 x 48]
//   D3 = DO [128 x 16] | weights
// TMEM (256 columns): working accumulator [0,64); weight-gradient
// accumulators persistent across the CTA's tiles:
//   dWc2^T [64,128)  dWc1 [128,176)  dW1d [176,208)  dWc3^T [208,224)  dW2d^T [224,240)
constexpr uint32_t kBufA = 9 * kChunk;  // 18432
constexpr uint32_t kBwdSmem = 3 * kBufA + 4 * kChunk + 6 * kChunk + 2 * kChunk + kWeightsBytes + 2 * kBiasTile64 +
                               kBiasTile16 + 128;
constexpr uint32_t kBwdTmemCols = 256;
constexpr int kColWc2 = 64, kColWc1 = 128, kColW1d = 176, kColWc3 = 208, kColW2d = 224;
constexpr int kColDX = 240;  // d(features) of the last tile, read by the scatter warps
// Warp specialisation: warps 0-3 run the MLP chain (one thread per tile row,
// thread 0 issues the MMAs), warps 4-7 run the hash-table scatter of the
// previous tile's d(features) from TMEM, so the L2-atomic-bound scatter
// overlaps the latency-bound MMA chain instead of extending it.
constexpr int kBwdThreads = 256;
#ifndef TFG_REGS_MLP
#define TFG_REGS_MLP 168
#endif
constexpr uint32_t kRegsMlp = TFG_REGS_MLP, kRegsScatter = 256 - TFG_REGS_MLP;  // 4 x 32 x 256 = 32768 per CTA

__device__ __forceinline__ void set_ones_chunk(uint8_t* buf, int chunk, int r) {
    float v[8] = {1.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    st_chunk(buf, r, chunk, v);
}

// Adds the CTA's TMEM weight-gradient accumulators into the global gradients.
// Row-major blocks whose rows are per-thread (dW1d, dWc1) go through a smem
// transpose so that their reds are coalesced (consecutive lanes, consecutive
// addresses: 4 sectors per warp instruction instead of 32); the MN-major
// blocks (dW2d^T, dWc2^T, dWc3^T) are coalesced as they come.  `scratch` is a
// free activation buffer; the 128 MLP threads call these together.
__device__ __forceinline__ void red_block_coalesced(float* __restrict__ g, const float* scratch, int n) {
    for (int j = threadIdx.x; j < n; j += kT) atomicAdd(g + j, scratch[j]);
}
__device__ __forceinline__ void flush_density(uint32_t tmem, float* __restrict__ gd, float* scratch) {
    int m = threadIdx.x;  // TMEM lane row
    float v[32];
    // dW1d [o=m][i] (cols 0..15), bias at col 16
    tld16(tmem, kColW1d, v);
    tld16(tmem, kColW1d + 16, v + 16);
    umma::ld_wait();
    if (m < kDHidden) {
#pragma unroll
        for (int i = 0; i < kFeatDim; ++i) scratch[m * kFeatDim + i] = v[i];
        atomicAdd(gd + kDB1 + m, v[16]);
    }
    asm volatile("bar.sync 1, 128;\n" ::: "memory");
    red_block_coalesced(gd + kDW1, scratch, kDHidden * kFeatDim);
    asm volatile("bar.sync 1, 128;\n" ::: "memory");  // scratch reused
    // dW2d^T [i=m][o], bias row m = 64
    tld16(tmem, kColW2d, v);
    umma::ld_wait();
    if (m < kDHidden)
        for (int o = 0; o < kDOut; ++o) atomicAdd(gd + kDW2 + o * kDHidden + m, v[o]);
    else if (m == kDHidden)
        for (int o = 0; o < kDOut; ++o) atomicAdd(gd + kDB2 + o, v[o]);
}
__device__ __forceinline__ void flush_color(uint32_t tmem, float* __restrict__ gc, float* scratch) {
    int m = threadIdx.x;
    float v[64];
    // dWc2^T [i=m][o], bias row 64
    tld16(tmem, kColWc2, v);
    tld16(tmem, kColWc2 + 16, v + 16);
    tld16(tmem, kColWc2 + 32, v + 32);
    tld16(tmem, kColWc2 + 48, v + 48);
    umma::ld_wait();
    if (m < kCHidden)
        for (int o = 0; o < kCHidden; ++o) atomicAdd(gc + kCW2 + o * kCHidden + m, v[o]);
    else if (m == kCHidden)
        for (int o = 0; o < kCHidden; ++o) atomicAdd(gc + kCB2 + o, v[o]);
    // dWc1 [o=m][i], i < 39, bias at col 39
    tld16(tmem, kColWc1, v);
    tld16(tmem, kColWc1 + 16, v + 16);
    tld16(tmem, kColWc1 + 32, v + 32);
    umma::ld_wait();
    if (m < kCHidden) {
        for (int i = 0; i < kCIn; ++i) scratch[m * kCIn + i] = v[i];
        atomicAdd(gc + kCB1 + m, v[kCIn]);
    }
    asm volatile("bar.sync 1, 128;\n" ::: "memory");
    red_block_coalesced(gc + kCW1, scratch, kCHidden * kCIn);
    asm volatile("bar.sync 1, 128;\n" ::: "memory");
    // dWc3^T [i=m][o], bias row 64
    tld16(tmem, kColWc3, v);
    umma::ld_wait();
    if (m < kCHidden)
        for (int o = 0; o < 3; ++o) atomicAdd(gc + kCW3 + o * kCHidden + m, v[o]);
    else if (m == kCHidden)
        for (int o = 0; o < 3; ++o) atomicAdd(gc + kCB3 + o, v[o]);
}

template <bool G>
__global__ void __launch_bounds__(kBwdThreads, 2) mlp_bwd_kernel(FieldArgs a, FieldGradArgs g,
                                                      const uint8_t* __restrict__ feat,
                                                      const int32_t* __restrict__ rays) {
    extern __shared__ __align__(128) uint8_t smem_raw[];
    __shared__ uint64_t bar_mma, bar_ld, bar_w, bar_e, bar_free;
    __shared__ uint32_t tmem_slot;
    uint8_t* p = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 127) & ~uintptr_t(127));
    uint8_t* H1 = carve(p, kBufA);
    uint8_t* C1 = carve(p, kBufA);
    uint8_t* C2 = carve(p, kBufA);
    uint8_t* X0 = carve(p, 4 * kChunk);
    uint8_t* CIN = carve(p, 6 * kChunk);
    uint8_t* D3 = carve(p, 2 * kChunk);
    uint8_t* DO = D3;  // D3 is dead once (A)'s MMAs have completed; DO is written in (C)
    Weights W = carve_weights(p);
    // bias tiles of the recomputed forward layers (as mlp_fwd_kernel: the
    // accumulators start at the bias, so both kernels compute the same
    // pre-activations bit for bit); the A side is X0's K step 1, whose
    // columns 16 and 17 are 1
    uint8_t* const bt_l1 = carve(p, kBiasTile64);
    uint8_t* const bt_l2 = carve(p, kBiasTile16);
    uint8_t* const bt_c2 = carve(p, kBiasTile64);
    const int r = threadIdx.x;
    if (r == 0) {
        umma::mbar_init(&bar_mma, 1);
        umma::mbar_init(&bar_ld, 1);
        umma::mbar_init(&bar_w, 1);
        umma::mbar_init(&bar_e, 1);
        umma::mbar_init(&bar_free, 4);
        umma::fence_mbar_init();
    }
    if (r < 32) umma::tmem_alloc<kBwdTmemCols>(&tmem_slot);
    if (r < kT) {
        stage_color(W, a.f.color);
        // constant ones chunks
        set_ones_chunk(H1, 8, r);
        set_ones_chunk(C1, 8, r);
        set_ones_chunk(C2, 8, r);
        const float o2[8] = {1.f, 1.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        st_chunk(X0, r, 2, o2);  // col 16: dW1d's bias column; 16-17: the bias MMAs' A
        float z[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        st_chunk(X0, r, 3, z);
        stage_bias_tile<64>(bt_c2, a.f.color + kCB2, kCHidden);
    }
    pdl_wait();  // the composite's gradients
    uint32_t n_tiles = a.status->n_tiles;
    sync_for_mma();
    const uint32_t tmem = tmem_slot;
    if (r >= kT) {
        // ================= scatter warps
        umma::reg_dealloc<kRegsScatter>();
        const int row = r - kT;
        const uint32_t quad = uint32_t(row >> 5);
        uint32_t ph_e = 0;
        for (uint32_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
            TileDesc td = a.tiles[t];
            bool live = row < td.n;
            float4 L = live ? a.s.local[uint64_t(td.start) + row] : make_float4(0.f, 0.f, 0.f, 0.f);
            umma::mbar_wait(&bar_e, ph_e);
            ph_e ^= 1u;
            umma::fence_after_sync();
            float v[16];
            umma::ld16(tmem + ((32u * quad) << 16) + uint32_t(kColDX), v);
            umma::ld_wait();
            umma::fence_before_sync();
            __syncwarp();
            if ((row & 31) == 0) umma::mbar_arrive(&bar_free);  // TMEM columns free again
            if constexpr (G)
                scatter_row_rt(a.hl, g.g_enc[td.slot], L.x, L.y, L.z, v, live);
            else
                scatter_row_bfly(g.g_enc[td.slot], L.x, L.y, L.z, v, live);
        }
        __syncthreads();  // pairs with the MLP warps' final barrier before tmem_free
        return;
    }
    umma::reg_alloc<kRegsMlp>();
    uint32_t ph_mma = 0, ph_ld = 0, ph_w = 0, ph_free = 0;
    int cur = -1;
    bool first_d = true, first_c = true, first_e = true;
    const uint32_t id64 = umma::idesc_bf16(128, 64, 0, 0);
    const uint32_t id16 = umma::idesc_bf16(128, 16, 0, 0);
    const uint32_t id64_kmn = umma::idesc_bf16(128, 64, 0, 1);  // A K-major, B MN-major
    const uint32_t id16_kmn = umma::idesc_bf16(128, 16, 0, 1);
    const uint32_t idw64 = umma::idesc_bf16(128, 64, 1, 1);     // weight grads: both MN-major
    const uint32_t idw48 = umma::idesc_bf16(128, 48, 1, 1);
    const uint32_t idw32 = umma::idesc_bf16(128, 32, 1, 1);
    const uint32_t idw16 = umma::idesc_bf16(128, 16, 1, 1);
    // the next tile's descriptor (packed) and ray ids one tile ahead, as in
    // mlp_fwd_kernel: this tile's sample and view-encoding loads then issue
    // without a dependent load in front of them
    const uint2* tiles2 = reinterpret_cast<const uint2*>(a.tiles);
    uint2 td_next = blockIdx.x < n_tiles ? __ldg(tiles2 + blockIdx.x) : make_uint2(0u, 0u);
    int ray_next = blockIdx.x < n_tiles ? rays[uint64_t(blockIdx.x) * kT + r] : -1;
    for (uint32_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
        asm volatile("" : "+r"(td_next.x), "+r"(td_next.y));
        const TileDesc td{td_next.x, uint16_t(td_next.y & 0xffffu), uint16_t(td_next.y >> 16)};
        const int ray = ray_next;
        if (t + gridDim.x < n_tiles) {
            td_next = __ldg(tiles2 + t + gridDim.x);
            ray_next = rays[uint64_t(t + gridDim.x) * kT + r];
        }
        if (td.slot != cur) {
            if (cur >= 0) flush_density(tmem, g.g_dnet[cur], reinterpret_cast<float*>(C1));
            stage_density(W, a.f.dnet[td.slot]);
            stage_bias_tile<64>(bt_l1, a.f.dnet[td.slot] + kDB1, kDHidden);
            stage_bias_tile<16>(bt_l2, a.f.dnet[td.slot] + kDB2, kDOut);
            cur = td.slot;
            first_d = true;
        }
        if (r == 0) {
            umma::mbar_expect_tx(&bar_ld, kFeatTile);
            umma::bulk_g2s(X0, feat + uint64_t(t) * kFeatTile, kFeatTile, &bar_ld);
        }
        bool live = r < td.n;
        float4 dio = live ? a.s.io[uint64_t(td.start) + r] : make_float4(0.f, 0.f, 0.f, 0.f);
        float ve[kViewDim];
        {
            const float4* v4 = a.venc + uint64_t(ray < 0 ? 0 : ray) * 6;
#pragma unroll
            for (int q = 0; q < 6; ++q) {
                float4 v = __ldg(v4 + q);
                ve[4 * q] = v.x;
                ve[4 * q + 1] = v.y;
                ve[4 * q + 2] = v.z;
                ve[4 * q + 3] = v.w;
            }
        }
        sync_mlp();
        umma::mbar_wait(&bar_ld, ph_ld);
        ph_ld ^= 1u;
        // ================= forward recompute
        if (r == 0) {
            umma::mma(tmem, kmaj(X0, kT, 1), kmaj(bt_l1, 64, 0), id64, 0);  // bias
            umma::mma(tmem, kmaj(X0, kT, 0), kmaj(W.w1d, kW1dRows, 0), id64, 1);
            umma::commit(&bar_mma);
        }
        wait_mma(&bar_mma, ph_mma);
        {
            float v[64];
            tld16(tmem, 0, v);
            tld16(tmem, 16, v + 16);
            tld16(tmem, 32, v + 32);
            tld16(tmem, 48, v + 48);
            umma::ld_wait();
#pragma unroll
            for (int c = 0; c < 8; ++c) st_chunk_relu(H1, r, c, v + 8 * c);
        }
        sync_mlp();
        if (r == 0) {
            umma::mma(tmem, kmaj(X0, kT, 1), kmaj(bt_l2, 16, 0), id16, 0);
#pragma unroll
            for (int k = 0; k < 4; ++k)
                umma::mma(tmem, kmaj(H1, kT, k), kmaj(W.w2d, kW2dRows, k), id16, 1);
            umma::commit(&bar_mma);
        }
        wait_mma(&bar_mma, ph_mma);
        {
            float v[16];
            tld16(tmem, 0, v);
            umma::ld_wait();
            float cin[48];
#pragma unroll
            for (int i = 0; i < kEmb; ++i) cin[i] = v[1 + i];
#pragma unroll
            for (int i = 0; i < kViewDim; ++i) cin[kEmb + i] = ve[i];
            cin[kCIn] = cin[kCIn + 1] = 1.f;  // bias columns (see stage_color)
#pragma unroll
            for (int i = kCIn + 2; i < 48; ++i) cin[i] = 0.f;
#pragma unroll
            for (int c = 0; c < 6; ++c) st_chunk(CIN, r, c, cin + 8 * c);
        }
        sync_mlp();
        if (r == 0) {
#pragma unroll
            for (int k = 0; k < 3; ++k)
                umma::mma(tmem, kmaj(CIN, kT, k), kmaj(W.wc1, kWc1Rows, k), id64, k > 0);
            umma::commit(&bar_mma);
        }
        wait_mma(&bar_mma, ph_mma);
        {
            float v[64];
            tld16(tmem, 0, v);
            tld16(tmem, 16, v + 16);
            tld16(tmem, 32, v + 32);
            tld16(tmem, 48, v + 48);
            umma::ld_wait();
#pragma unroll
            for (int c = 0; c < 8; ++c) st_chunk_relu(C1, r, c, v + 8 * c);
        }
        sync_mlp();
        if (r == 0) {
            umma::mma(tmem, kmaj(X0, kT, 1), kmaj(bt_c2, 64, 0), id64, 0);
#pragma unroll
            for (int k = 0; k < 4; ++k)
                umma::mma(tmem, kmaj(C1, kT, k), kmaj(W.wc2, kWc2Rows, k), id64, 1);
            umma::commit(&bar_mma);
        }
        wait_mma(&bar_mma, ph_mma);
        {
            float v[64];
            tld16(tmem, 0, v);
            tld16(tmem, 16, v + 16);
            tld16(tmem, 32, v + 32);
            tld16(tmem, 48, v + 48);
            umma::ld_wait();
#pragma unroll
            for (int c = 0; c < 8; ++c) st_chunk_relu(C2, r, c, v + 8 * c);
        }
        {
            // K3 already applied the sigmoid derivative: io = (d raw sigma,
            // d pre-sigmoid r, g, b), so the colour output layer is not
            // recomputed.  (D3 = DO: the previous tile's readers of DO have
            // completed; one barrier covers C2 and D3.)
            float d3[16];
            d3[0] = dio.y;
            d3[1] = dio.z;
            d3[2] = dio.w;
#pragma unroll
            for (int o = 3; o < 16; ++o) d3[o] = 0.f;
            st_chunk(D3, r, 0, d3);
            st_chunk(D3, r, 1, d3 + 8);
        }
        sync_mlp();
        // ================= backward
        // (A) dC2pre = D3 . Wc3 ; dWc3^T += [C2|1]^T . D3
        if (r == 0) {
            umma::mma(tmem, kmaj(D3, kT, 0), mnmaj(W.wc3, kWc3Rows, 0), id64_kmn, 0);
            umma::commit(&bar_mma);
#pragma unroll
            for (int k = 0; k < 8; ++k)
                umma::mma(tmem + kColWc3, mnmaj(C2, kT, k), mnmaj(D3, kT, k), idw16, (first_c && k == 0) ? 0 : 1);
            umma::commit(&bar_w);
        }
        wait_mma(&bar_mma, ph_mma);
        {
            float v[64];
            tld16(tmem, 0, v);
            tld16(tmem, 16, v + 16);
            tld16(tmem, 32, v + 32);
            tld16(tmem, 48, v + 48);
            umma::ld_wait();
            wait_mma(&bar_w, ph_w);  // dWc3^T has read C2
#pragma unroll
            for (int c = 0; c < 8; ++c) st_chunk_masked(C2, r, c, v + 8 * c);  // DC2 over C2
        }
        sync_mlp();
        // (B) dC1pre = DC2 . Wc2 ; dWc2^T += [C1|1]^T . DC2
        if (r == 0) {
#pragma unroll
            for (int k = 0; k < 4; ++k)
                umma::mma(tmem, kmaj(C2, kT, k), mnmaj(W.wc2, kWc2Rows, k), id64_kmn, k > 0);
            umma::commit(&bar_mma);
#pragma unroll
            for (int k = 0; k < 8; ++k)
                umma::mma(tmem + kColWc2, mnmaj(C1, kT, k), mnmaj(C2, kT, k), idw64, (first_c && k == 0) ? 0 : 1);
            umma::commit(&bar_w);
        }
        wait_mma(&bar_mma, ph_mma);
        {
            float v[64];
            tld16(tmem, 0, v);
            tld16(tmem, 16, v + 16);
            tld16(tmem, 32, v + 32);
            tld16(tmem, 48, v + 48);
            umma::ld_wait();
            wait_mma(&bar_w, ph_w);  // dWc2^T has read C1
#pragma unroll
            for (int c = 0; c < 8; ++c) st_chunk_masked(C1, r, c, v + 8 * c);  // DC1 over C1
        }
        sync_mlp();
        // (C) dCIN[0:16] = DC1 . Wc1[:, 0:16] ; dWc1 += DC1^T . CIN
        if (r == 0) {
#pragma unroll
            for (int k = 0; k < 4; ++k)
                umma::mma(tmem, kmaj(C1, kT, k), mnmaj(W.wc1, kWc1Rows, k), id16_kmn, k > 0);
            umma::commit(&bar_mma);
#pragma unroll
            for (int k = 0; k < 8; ++k)
                umma::mma(tmem + kColWc1, mnmaj(C1, kT, k), mnmaj(CIN, kT, k), idw48, (first_c && k == 0) ? 0 : 1);
            umma::commit(&bar_w);
        }
        wait_mma(&bar_mma, ph_mma);
        first_c = false;
        {
            float v[16];
            tld16(tmem, 0, v);
            umma::ld_wait();
            float d[16];
            d[0] = dio.x;  // d raw sigma (K3)
#pragma unroll
            for (int i = 0; i < kEmb; ++i) d[1 + i] = v[i];
            wait_mma(&bar_w, ph_w);  // (in-order retire; keeps the phases paired)
            st_chunk(DO, r, 0, d);
            st_chunk(DO, r, 1, d + 8);
        }
        sync_mlp();
        // (D) dH1pre = DO . W2d ; dW2d^T += [H1|1]^T . DO
        if (r == 0) {
            umma::mma(tmem, kmaj(DO, kT, 0), mnmaj(W.w2d, kW2dRows, 0), id64_kmn, 0);
            umma::commit(&bar_mma);
#pragma unroll
            for (int k = 0; k < 8; ++k)
                umma::mma(tmem + kColW2d, mnmaj(H1, kT, k), mnmaj(DO, kT, k), idw16, (first_d && k == 0) ? 0 : 1);
            umma::commit(&bar_w);
        }
        wait_mma(&bar_mma, ph_mma);
        {
            float v[64];
            tld16(tmem, 0, v);
            tld16(tmem, 16, v + 16);
            tld16(tmem, 32, v + 32);
            tld16(tmem, 48, v + 48);
            umma::ld_wait();
            wait_mma(&bar_w, ph_w);  // dW2d^T has read H1
#pragma unroll
            for (int c = 0; c < 8; ++c) st_chunk_masked(H1, r, c, v + 8 * c);  // DH1 over H1
        }
        sync_mlp();
        // (E) dX0 = DH1 . W1d into the scatter warps' columns (once they have
        // read the previous tile's) ; dW1d += DH1^T . [X0|1|0]
        if (r == 0) {
            if (!first_e) {
                umma::mbar_wait(&bar_free, ph_free);
                ph_free ^= 1u;
                umma::fence_after_sync();
            }
#pragma unroll
            for (int k = 0; k < 4; ++k)
                umma::mma(tmem + kColDX, kmaj(H1, kT, k), mnmaj(W.w1d, kW1dRows, k), id16_kmn, k > 0);
            umma::commit(&bar_e);
#pragma unroll
            for (int k = 0; k < 8; ++k)
                umma::mma(tmem + kColW1d, mnmaj(H1, kT, k), mnmaj(X0, kT, k), idw32, (first_d && k == 0) ? 0 : 1);
            umma::commit(&bar_w);
        }
        first_d = false;
        first_e = false;
        wait_mma(&bar_w, ph_w);  // dW1d has read H1 / X0 before the next tile
    }
    umma::fence_before_sync();
    asm volatile("bar.sync 1, 128;\n" ::: "memory");
    umma::fence_after_sync();
    if (cur >= 0) flush_density(tmem, g.g_dnet[cur], reinterpret_cast<float*>(C1));
    if (!first_c) flush_color(tmem, g.g_color, reinterpret_cast<float*>(C1));
    umma::fence_before_sync();
    __syncthreads();
    if (r < 32) umma::tmem_free<kBwdTmemCols>(tmem);
}

// ------------------------------------------------------------------ launchers
// Function attributes belong to the current device's context: set them once
// per device (not once per process), under a lock so that no launch on that
// device overtakes the setting.
static void set_smem_attributes_once() {
    static std::mutex mu;
    static uint64_t done = 0;
    int dev = 0;
    cudaGetDevice(&dev);
    const uint64_t bit = uint64_t(1) << (dev & 63);
    std::lock_guard<std::mutex> lock(mu);
    if (done & bit) return;
    cudaFuncSetAttribute(mlp_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kFwdSmem));

    cudaFuncSetAttribute(mlp_bwd_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kBwdSmem));
    cudaFuncSetAttribute(mlp_bwd_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kBwdSmem));
    done |= bit;
}

void launch_field_forward_tc(const FieldArgs& a, uint8_t* feat, int32_t* rays, int sms,
                             cudaStream_t st, uint64_t* launches) {
    set_smem_attributes_once();
#ifndef TFG_GATHER_CTAS
#define TFG_GATHER_CTAS 6  // r2 (fp16 tables, final MLP): 4: 0.535, 5: 0.511, 6: 0.507, 7: 0.513, 8: 0.517 ms field_fwd
#endif
#ifndef TFG_MLPF_CTAS
#define TFG_MLPF_CTAS 4
#endif
    if (a.hl.generic)
        launch_pdl(hash_fwd_kernel<true>, dim3(sms * TFG_GATHER_CTAS), dim3(128), 0, st, a, feat, rays);
    else
        launch_pdl(hash_fwd_kernel<false>, dim3(sms * TFG_GATHER_CTAS), dim3(128), 0, st, a, feat, rays);
    launch_pdl(mlp_fwd_kernel, dim3(sms * TFG_MLPF_CTAS), dim3(128), kFwdSmem, st, a, feat, rays);  // 4 per SM
    *launches += 2;
}

void launch_field_backward_tc(const FieldArgs& a, const FieldGradArgs& g, uint8_t* feat,
                              int32_t* rays, int sms, cudaStream_t st, uint64_t* launches) {
    set_smem_attributes_once();
    // the feature tiles of the forward pass (same batch) are still resident;
    // the hash-table scatter is fused into the backward's last epilogue
    if (a.hl.generic)
        launch_pdl(mlp_bwd_kernel<true>, dim3(sms * 2), dim3(kBwdThreads), kBwdSmem, st, a, g, feat, rays);
    else
        launch_pdl(mlp_bwd_kernel<false>, dim3(sms * 2), dim3(kBwdThreads), kBwdSmem, st, a, g, feat, rays);
    *launches += 1;
}

} // namespace tfg
