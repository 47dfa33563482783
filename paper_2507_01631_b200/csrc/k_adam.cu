// k_adam.cu — K5: fused Adam over the window's parameter groups (4 x enc,
// 4 x dnet, colour) in one launch (adam_step, field.hpp:45-48).
// Compiled with -fmad=false so the update rounds exactly like the reference
// formula (bit-identical to the oracle for identical gradients):
//   m = b1 m + (1-b1) g;  v = b2 v + (1-b2) g^2;
//   p = p - lr * (m / bc1) / (sqrt(v / bc2) + eps)
// with lr and bias corrections of the persistent per-group step count
// computed on the host.  A group with a non-finite gradient aborts the whole
// step (the reference throws before updating, naming the group).
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "tf_common.cuh"
#include "tf_kernels.h"

namespace tfg {

__device__ __forceinline__ int group_of(const AdamArgs& a, uint64_t i) {
    int g = 0;
    while (g + 1 < a.n_groups && i >= a.g[g + 1].offset) ++g;
    return g;
}

// Both kernels stream float4s: every group offset is a multiple of 4
// (tfg_optimizer_step checks), so a float4 never straddles two groups; the
// last total % 4 elements go one by one.
__global__ void __launch_bounds__(256) grad_check_kernel(AdamArgs a, uint64_t total) {
    pdl_wait();
    uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    uint32_t bad = 0;  // bitmask of groups
    const uint64_t n4 = total >> 2;
    const float4* g4 = reinterpret_cast<const float4*>(a.grads);
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n4; i += stride) {
        float4 g = g4[i];
        if (!(isfinite(g.x) && isfinite(g.y) && isfinite(g.z) && isfinite(g.w))) bad |= 1u << group_of(a, 4 * i);
    }
    for (uint64_t i = 4 * n4 + uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += stride) {
        float g = a.grads[i];
        if (!isfinite(g)) bad |= 1u << group_of(a, i);
    }
    bad = __reduce_or_sync(0xffffffffu, bad);
    if ((threadIdx.x & 31) == 0 && bad) {
        for (int g = 0; g < a.n_groups; ++g)
            if (bad & (1u << g)) atomicOr(&a.group_flags[g], 1u);
    }
}

__global__ void __launch_bounds__(256) adam_kernel(AdamArgs a, uint64_t total) {
    pdl_wait();
    __shared__ int skip;
    if (threadIdx.x == 0) {
        int s = 0;
        for (int g = 0; g < a.n_groups; ++g) s |= a.group_flags[g] ? 1 : 0;
        // an earlier step's non-finite error not yet read by the host: the
        // reference would have thrown, so no later step is applied either
        const int pending = a.sticky[0] != 0;
        skip = s | pending;
        if (s && !pending && blockIdx.x == 0) {
            for (int g = 0; g < a.n_groups; ++g)
                if (a.group_flags[g]) {
                    a.sticky[1] = uint32_t(g);
                    break;
                }
            a.sticky[2] = a.seq;
            __threadfence();
            a.sticky[0] = 1u;
        }
    }
    __syncthreads();
    if (skip) return;
    uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    // the update of one element (adam_step's formula and rounding)
    auto upd = [&](const AdamGroup& G, float g, float& m, float& v, float& p) {
        m = a.beta1 * m + a.omb1 * g;
        v = a.beta2 * v + a.omb2 * (g * g);
        float mh = m / G.bc1;
        float vh = v / G.bc2;
        p = p - G.lr * mh / (sqrtf(vh) + a.eps);
    };
    const uint64_t n4 = total >> 2;
    const float4* g4 = reinterpret_cast<const float4*>(a.grads);
    float4* m4 = reinterpret_cast<float4*>(a.m);
    float4* v4 = reinterpret_cast<float4*>(a.v);
    float4* p4 = reinterpret_cast<float4*>(a.params);
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n4; i += stride) {
        const AdamGroup& G = a.g[group_of(a, 4 * i)];
        const float4 g = g4[i];
        float4 m = m4[i], v = v4[i], p = p4[i];
        upd(G, g.x, m.x, v.x, p.x);
        upd(G, g.y, m.y, v.y, p.y);
        upd(G, g.z, m.z, v.z, p.z);
        upd(G, g.w, m.w, v.w, p.w);
        m4[i] = m;
        v4[i] = v;
        p4[i] = p;
        if (G.half_slot >= 0) {  // the slot's fp16 table shadow (forward gather)
            __half2* h = reinterpret_cast<__half2*>(a.enc16) + (uint64_t(G.half_slot) * a.enc16_stride + (4 * i - G.offset)) / 2;
            uint2 q;
            __half2 lo = __floats2half2_rn(p.x, p.y), hi = __floats2half2_rn(p.z, p.w);
            q.x = *reinterpret_cast<uint32_t*>(&lo);
            q.y = *reinterpret_cast<uint32_t*>(&hi);
            *reinterpret_cast<uint2*>(h) = q;
        }
    }
    for (uint64_t i = 4 * n4 + uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += stride) {
        const AdamGroup& G = a.g[group_of(a, i)];
        float m = a.m[i], v = a.v[i], p = a.params[i];
        upd(G, a.grads[i], m, v, p);
        a.m[i] = m;
        a.v[i] = v;
        a.params[i] = p;
        if (G.half_slot >= 0)
            reinterpret_cast<__half*>(a.enc16)[uint64_t(G.half_slot) * a.enc16_stride + (i - G.offset)] = __float2half_rn(p);
    }
}

__global__ void __launch_bounds__(256) enc_half_kernel(const float* __restrict__ params, uint64_t stride,
                                                       uint64_t enc_n, uint64_t out_stride,
                                                       __half2* __restrict__ out) {
    pdl_wait();
    const int k = blockIdx.y;
    const float2* src = reinterpret_cast<const float2*>(params + uint64_t(k) * stride);
    __half2* dst = out + uint64_t(k) * out_stride / 2;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < enc_n / 2; i += uint64_t(gridDim.x) * blockDim.x)
        dst[i] = __float22half2_rn(src[i]);
}

void launch_enc_half(const float* params, uint64_t stride, int n, uint64_t enc_n, uint64_t out_stride, void* out,
                     cudaStream_t st, uint64_t* launches) {
    launch_pdl(enc_half_kernel, dim3(148, n), dim3(256), 0, st, params, stride, enc_n, out_stride,
               static_cast<__half2*>(out));
    *launches += 1;
}

void launch_adam(const AdamArgs& a, uint64_t total, cudaStream_t st, uint64_t* launches) {
    int blocks = int((total / 4 + 255) / 256);
    if (blocks < 1) blocks = 1;
    if (blocks > 148 * 8) blocks = 148 * 8;
    launch_pdl(grad_check_kernel, dim3(blocks), dim3(256), 0, st, a, total);
    launch_pdl(adam_kernel, dim3(blocks), dim3(256), 0, st, a, total);
    *launches += 2;
}

} // namespace tfg
