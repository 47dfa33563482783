// tf_hash.cuh — multi-resolution hash-grid gather / scatter shared by the
// field kernels (HashGridT, nn.hpp:199-266).
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "tf_common.cuh"
#include "tf_kernels.h"

namespace tfg {

// HashGridT::lookup_p (nn.hpp:213-228): clamp, scale, cell + fraction,
// 8 trilinear corners; dense indexing when (N+1)^3 <= T, else spatial hash.
struct Corner {
    uint32_t idx[8];
    float w[8];
};

// Level layout of the default FieldConfig (nn.hpp:14-45: N_min 16, N_max 256,
// 8 levels, T = 2^15): resolutions, entry offsets; levels 0-1 are dense.
// tfg_create compares the runtime HashLayout with these constants and sets
// HashLayout::generic when they differ (the kernels' runtime-layout
// instantiations then run).
__host__ __device__ constexpr int level_res_c(int l) {
    return l == 0 ? 16 : l == 1 ? 24 : l == 2 ? 35 : l == 3 ? 53 : l == 4 ? 78 : l == 5 ? 116 : l == 6 ? 172 : 256;
}
__host__ __device__ constexpr uint32_t level_off_c(int l) {
    return l == 0 ? 0u : l == 1 ? 4913u : l == 2 ? 20538u : l == 3 ? 53306u : l == 4 ? 86074u
         : l == 5 ? 118842u : l == 6 ? 151610u : 184378u;
}

// HashGridT::cell_of + corner_entry (nn.hpp:248-266) for level L, with the
// level constants folded: clamp to [0,1], scale, cell + fraction, 8 trilinear
// weights ((wx*wy)*wz, the reference's product order) and entry indices
// (dense x + n(y + n z), or the spatial hash x ^ y*2654435761 ^ z*805459861).
template <int L>
__device__ __forceinline__ void hash_level_c(float x, float y, float z, Corner& c) {
    constexpr int n = level_res_c(L);
    constexpr uint32_t n1 = uint32_t(n + 1);
    constexpr bool dense = uint64_t(n1) * n1 * n1 <= uint64_t(kTable);
    float p[3] = {x, y, z};
    int q[3];
    float f[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        float v = fminf(fmaxf(p[k], 0.f), 1.f);
        float sc = v * float(n);
        int ci = int(sc);
        ci = ci > n - 1 ? n - 1 : ci;
        q[k] = ci;
        f[k] = sc - float(ci);
    }
    float wx[2] = {1.f - f[0], f[0]}, wy[2] = {1.f - f[1], f[1]}, wz[2] = {1.f - f[2], f[2]};
    float wxy[4] = {wx[0] * wy[0], wx[1] * wy[0], wx[0] * wy[1], wx[1] * wy[1]};
#pragma unroll
    for (int k = 0; k < 8; ++k) c.w[k] = wxy[k & 3] * wz[k >> 2];
    if constexpr (dense) {
        uint32_t base = level_off_c(L) + uint32_t(q[0]) + n1 * (uint32_t(q[1]) + n1 * uint32_t(q[2]));
#pragma unroll
        for (int k = 0; k < 8; ++k)
            c.idx[k] = base + uint32_t(k & 1) + n1 * uint32_t((k >> 1) & 1) + n1 * n1 * uint32_t(k >> 2);
    } else {
        uint32_t X = uint32_t(q[0]);
        uint32_t hy0 = uint32_t(q[1]) * 2654435761u, hy1 = hy0 + 2654435761u;
        uint32_t hz0 = uint32_t(q[2]) * 805459861u, hz1 = hz0 + 805459861u;
        uint32_t hyz[4] = {hy0 ^ hz0, hy1 ^ hz0, hy0 ^ hz1, hy1 ^ hz1};
#pragma unroll
        for (int k = 0; k < 8; ++k)
            c.idx[k] = level_off_c(L) + (((X + uint32_t(k & 1)) ^ hyz[k >> 1]) & uint32_t(kTable - 1));
    }
}

// The same for a layout read at run time (a non-default n_min / n_max /
// table_size): identical arithmetic with the level constants loaded.
__device__ __forceinline__ void hash_level_rt(const HashLayout& hl, int l, float x, float y, float z,
                                              Corner& c) {
    const int n = hl.res[l];
    const uint32_t n1 = uint32_t(n + 1), off = hl.off[l];
    float p[3] = {x, y, z};
    int q[3];
    float f[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        float v = fminf(fmaxf(p[k], 0.f), 1.f);
        float sc = v * float(n);
        int ci = int(sc);
        ci = ci > n - 1 ? n - 1 : ci;
        q[k] = ci;
        f[k] = sc - float(ci);
    }
    float wx[2] = {1.f - f[0], f[0]}, wy[2] = {1.f - f[1], f[1]}, wz[2] = {1.f - f[2], f[2]};
    float wxy[4] = {wx[0] * wy[0], wx[1] * wy[0], wx[0] * wy[1], wx[1] * wy[1]};
#pragma unroll
    for (int k = 0; k < 8; ++k) c.w[k] = wxy[k & 3] * wz[k >> 2];
    if (hl.dense[l]) {
        uint32_t base = off + uint32_t(q[0]) + n1 * (uint32_t(q[1]) + n1 * uint32_t(q[2]));
#pragma unroll
        for (int k = 0; k < 8; ++k)
            c.idx[k] = base + uint32_t(k & 1) + n1 * uint32_t((k >> 1) & 1) + n1 * n1 * uint32_t(k >> 2);
    } else {
        uint32_t X = uint32_t(q[0]);
        uint32_t hy0 = uint32_t(q[1]) * 2654435761u, hy1 = hy0 + 2654435761u;
        uint32_t hz0 = uint32_t(q[2]) * 805459861u, hz1 = hz0 + 805459861u;
        uint32_t hyz[4] = {hy0 ^ hz0, hy1 ^ hz0, hy0 ^ hz1, hy1 ^ hz1};
#pragma unroll
        for (int k = 0; k < 8; ++k) c.idx[k] = off + (((X + uint32_t(k & 1)) ^ hyz[k >> 1]) & hl.mask);
    }
}

// Level l of the layout: folded constants (G = false) or read at run time.
template <bool G>
__device__ __forceinline__ void hash_level(const HashLayout& hl, int l, float x, float y, float z,
                                           Corner& c) {
    if constexpr (G) {
        hash_level_rt(hl, l, x, y, z, c);
    } else {
        switch (l) {
        case 0: hash_level_c<0>(x, y, z, c); break;
        case 1: hash_level_c<1>(x, y, z, c); break;
        case 2: hash_level_c<2>(x, y, z, c); break;
        case 3: hash_level_c<3>(x, y, z, c); break;
        case 4: hash_level_c<4>(x, y, z, c); break;
        case 5: hash_level_c<5>(x, y, z, c); break;
        case 6: hash_level_c<6>(x, y, z, c); break;
        default: hash_level_c<7>(x, y, z, c); break;
        }
    }
}

// The two x-neighbour corners (dx = 0, 1) of a cell hit the same aligned
// 16-byte entry pair whenever idx1 == idx0 ^ 1 (dense levels: even index;
// hashed levels: even cell x, since (x + 1) ^ h = (x ^ h) ^ 1).  Such pairs
// are fetched with one 16-byte load (fewer L1 wavefronts).
template <bool G>
__device__ __forceinline__ void hash_encode(const HashLayout& hl, const float* __restrict__ tab,
                                            float x, float y, float z, float* feat) {
    const float2* t2 = reinterpret_cast<const float2*>(tab);
    const float4* t4 = reinterpret_cast<const float4*>(tab);
#pragma unroll
    for (int l = 0; l < kLevels; ++l) {
        Corner c;
        hash_level<G>(hl, l, x, y, z, c);
        float2 e[8];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            uint32_t i0 = c.idx[2 * q], i1 = c.idx[2 * q + 1];
            if (i1 == (i0 ^ 1u)) {
                float4 v = __ldg(t4 + (i0 >> 1));
                bool odd = i0 & 1u;
                e[2 * q] = odd ? make_float2(v.z, v.w) : make_float2(v.x, v.y);
                e[2 * q + 1] = odd ? make_float2(v.x, v.y) : make_float2(v.z, v.w);
            } else {
                e[2 * q] = __ldg(t2 + i0);
                e[2 * q + 1] = __ldg(t2 + i1);
            }
        }
        float a0 = 0.f, a1 = 0.f;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            a0 += c.w[k] * e[k].x;
            a1 += c.w[k] * e[k].y;
        }
        feat[2 * l] = a0;
        feat[2 * l + 1] = a1;
    }
}

// The same gather from the fp16 shadow tables: an entry is one __half2
// (4 bytes), an aligned x-neighbour pair one 8-byte load; the weights and
// the sums stay fp32.  Half the bytes of hash_encode returned to registers.
template <bool G>
__device__ __forceinline__ void hash_encode16(const HashLayout& hl, const void* __restrict__ tab,
                                              float x, float y, float z, float* feat) {
    const __half2* t2 = reinterpret_cast<const __half2*>(tab);
    const uint2* t4 = reinterpret_cast<const uint2*>(tab);
#pragma unroll
    for (int l = 0; l < kLevels; ++l) {
        Corner c;
        hash_level<G>(hl, l, x, y, z, c);
        float2 e[8];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            uint32_t i0 = c.idx[2 * q], i1 = c.idx[2 * q + 1];
            if (i1 == (i0 ^ 1u)) {
                const uint2 v = __ldg(t4 + (i0 >> 1));
                const float2 lo = __half22float2(*reinterpret_cast<const __half2*>(&v.x));
                const float2 hi = __half22float2(*reinterpret_cast<const __half2*>(&v.y));
                bool odd = i0 & 1u;
                e[2 * q] = odd ? hi : lo;
                e[2 * q + 1] = odd ? lo : hi;
            } else {
                e[2 * q] = __half22float2(__ldg(t2 + i0));
                e[2 * q + 1] = __half22float2(__ldg(t2 + i1));
            }
        }
        float a0 = 0.f, a1 = 0.f;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            a0 += c.w[k] * e[k].x;
            a1 += c.w[k] * e[k].y;
        }
        feat[2 * l] = a0;
        feat[2 * l + 1] = a1;
    }
}

} // namespace tfg
