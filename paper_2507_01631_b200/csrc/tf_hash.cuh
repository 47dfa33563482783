// tf_hash.cuh — multi-resolution hash-grid gather / scatter shared by the
// field kernels (HashGridT, nn.hpp:199-266).
#pragma once

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
__device__ __forceinline__ void hash_level(const HashLayout& hl, int l, float x, float y, float z,
                                           Corner& c) {
    int n = hl.res[l];
    float p[3] = {x, y, z};
    int ci[3];
    float f[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        float v = p[k];
        v = v < 0.f ? 0.f : v;
        v = v > 1.f ? 1.f : v;
        float sc = v * float(n);
        int q = int(sc);
        q = q > n - 1 ? n - 1 : q;
        ci[k] = q;
        f[k] = sc - float(q);
    }
    uint32_t np1 = uint32_t(n + 1);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        int dx = k & 1, dy = (k >> 1) & 1, dz = (k >> 2) & 1;
        c.w[k] = (dx ? f[0] : 1.f - f[0]) * (dy ? f[1] : 1.f - f[1]) * (dz ? f[2] : 1.f - f[2]);
        uint32_t X = uint32_t(ci[0] + dx), Y = uint32_t(ci[1] + dy), Z = uint32_t(ci[2] + dz);
        uint32_t e = hl.dense[l] ? X + np1 * (Y + np1 * Z)
                                 : ((X ^ (Y * 2654435761u) ^ (Z * 805459861u)) & uint32_t(kTable - 1));
        c.idx[k] = hl.off[l] + e;
    }
}

// The two x-neighbour corners (dx = 0, 1) of a cell hit the same aligned
// 16-byte entry pair whenever idx1 == idx0 ^ 1 (dense levels: even index;
// hashed levels: even cell x, since (x + 1) ^ h = (x ^ h) ^ 1).  Such pairs
// are fetched with one 16-byte load (fewer L1 wavefronts).
__device__ __forceinline__ void hash_encode(const HashLayout& hl, const float* __restrict__ tab,
                                            float x, float y, float z, float* feat) {
    const float2* t2 = reinterpret_cast<const float2*>(tab);
    const float4* t4 = reinterpret_cast<const float4*>(tab);
#pragma unroll
    for (int l = 0; l < kLevels; ++l) {
        Corner c;
        hash_level(hl, l, x, y, z, c);
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

__device__ __forceinline__ void hash_scatter(const HashLayout& hl, float* __restrict__ g, float x,
                                             float y, float z, const float* d) {
    float2* g2 = reinterpret_cast<float2*>(g);
#pragma unroll
    for (int l = 0; l < kLevels; ++l) {
        Corner c;
        hash_level(hl, l, x, y, z, c);
#pragma unroll
        for (int k = 0; k < 8; ++k)
            atomicAdd(g2 + c.idx[k], make_float2(c.w[k] * d[2 * l], c.w[k] * d[2 * l + 1]));
    }
}

} // namespace tfg
