// k_field.cu — K6: the occupancy update, TileField::update_occupancy
// (field.hpp:100-102).  4 x 32^3 density probes per update
// (every 16 iterations): hash gather + density MLP on CUDA cores in fp32,
// weights in shared memory.  The training-path field (K2/K4) is k_field_tc.cu.
#include <cuda_runtime.h>

#include "tf_common.cuh"
#include "tf_hash.cuh"
#include "tf_kernels.h"

namespace tfg {

__device__ __forceinline__ void load_floats(float* dst, const float* __restrict__ src, int n) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];
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
    if (a.update && !(a.sticky && a.sticky[0])) {
        int x = v % kOccRes, y = (v / kOccRes) % kOccRes, z = v / (kOccRes * kOccRes);
        Rng rng(hash_combine(a.base_key[slot], uint64_t(v)));
        float ux = rng.flt(), uy = rng.flt(), uz = rng.flt();
        float px = (float(x) + ux) / float(kOccRes);
        float py = (float(y) + uy) / float(kOccRes);
        float pz = (float(z) + uz) / float(kOccRes);
        float feat[kFeatDim];
        if (a.hl.generic)
            hash_encode<true>(a.hl, a.enc[slot], px, py, pz, feat);
        else
            hash_encode<false>(a.hl, a.enc[slot], px, py, pz, feat);
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
