// red_peak.cu — microbenchmark of the resource that bounds the field
// backward's hash-gradient scatter: `red.global.add` of fp32 vectors at
// random indices into a table the size of the window's hash tables (4 tiles x
// 434,292 floats = 6.9 MB, L2-resident).  Every lane of a warp targets an
// independent random entry, as in mlp_bwd_kernel's scatter warps (one sample
// per lane).  Prints one JSON object: the best payload GB/s over the variants
// (v2 = float2 per red, v4 = float4 per red, f32 = scalar) and grid sizes.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o red_peak tools/red_peak.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdint>
#include <vector>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16;
    x *= 0x7feb352dU;
    x ^= x >> 15;
    x *= 0x846ca68bU;
    x ^= x >> 16;
    return x;
}

template <int kVec>
__global__ void __launch_bounds__(256) red_kernel(float* __restrict__ table, uint32_t n_entries, int iters,
                                                  uint32_t seed) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t h = hash32(t ^ seed);
    const float v = 1e-7f;
#pragma unroll 4
    for (int i = 0; i < iters; ++i) {
        h = hash32(h + 0x9e3779b9U);
        const uint32_t e = h % n_entries;
        float* p = table + uint64_t(e) * kVec;
        if constexpr (kVec == 4) {
            asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v), "f"(v), "f"(v), "f"(v)
                         : "memory");
        } else if constexpr (kVec == 2) {
            asm volatile("red.global.add.v2.f32 [%0], {%1, %2};" ::"l"(p), "f"(v), "f"(v) : "memory");
        } else {
            asm volatile("red.global.add.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
        }
    }
}

template <int kVec>
double run(float* table, uint32_t floats, int blocks, int iters) {
    const uint32_t n_entries = floats / kVec;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    red_kernel<kVec><<<blocks, 256>>>(table, n_entries, iters, 1);  // warm-up
    cudaEventRecord(a);
    const int reps = 5;
    for (int r = 0; r < reps; ++r) red_kernel<kVec><<<blocks, 256>>>(table, n_entries, iters, 7 + r);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    const double bytes = double(reps) * blocks * 256.0 * iters * kVec * 4.0;
    return bytes / (ms / 1e3) / 1e9;
}

int main() {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceProp prop;
    cudaGetDeviceProperties(&prop, dev);
    const uint32_t floats = 4u * 434292u;  // the window's hash tables
    float* table = nullptr;
    if (cudaMalloc(&table, size_t(floats) * 4) != cudaSuccess) return 1;
    cudaMemset(table, 0, size_t(floats) * 4);
    const int iters = 256;
    double best = 0.0;
    const char* best_name = "";
    int best_blocks = 0;
    std::printf("{\"gpu\": \"%s\", \"sms\": %d, \"table_bytes\": %u, \"variants\": [", prop.name, sms, floats * 4);
    bool first = true;
    for (int per_sm : {4, 8, 16}) {
        const int blocks = sms * per_sm;
        double g[3] = {run<1>(table, floats, blocks, iters), run<2>(table, floats, blocks, iters),
                       run<4>(table, floats, blocks, iters)};
        const char* nm[3] = {"f32", "v2", "v4"};
        for (int k = 0; k < 3; ++k) {
            std::printf("%s{\"op\": \"red.global.add.%s\", \"blocks\": %d, \"GBps\": %.1f}", first ? "" : ", ",
                        k == 0 ? "f32" : (k == 1 ? "v2.f32" : "v4.f32"), blocks, g[k]);
            first = false;
            if (g[k] > best) {
                best = g[k];
                best_name = nm[k];
                best_blocks = blocks;
            }
        }
    }
    cudaError_t e = cudaDeviceSynchronize();
    std::printf("], \"best_GBps\": %.1f, \"best_variant\": \"%s\", \"best_blocks\": %d, \"status\": \"%s\", "
                "\"source\": \"tools/red_peak.cu: random-index red.global.add into a 6.9 MB table, "
                "one independent entry per lane, CUDA events, best of variants\"}\n",
                best, best_name, best_blocks, cudaGetErrorString(e));
    cudaFree(table);
    return e == cudaSuccess ? 0 : 1;
}
