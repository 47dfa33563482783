// umma_probe.cu — hardware check of the tcgen05 operand conventions used by
// the field kernels (paper_2507_01631_b200/csrc/umma.cuh): K-major and
// MN-major bf16 operands in the chunk-major interleave layout, fp32 TMEM
// accumulation, tcgen05.ld readback.  Prints max errors; exit 0 iff all pass.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../../paper_2507_01631_b200/csrc/umma.cuh"

using namespace tfg;

// Case: D[M=128 x N] = sum_k A(m,k) B(k,n), with A given as a stored tile
// (rows x cols) read K-major (rows=M, cols=K) or MN-major (rows=K, cols=M),
// and B given as (rows x cols) read K-major (rows=N, cols=K) or MN-major
// (rows=K, cols=N).
struct Case {
    int N, K;
    int a_mn, b_mn;
};

__global__ void probe(const __nv_bfloat16* gA, int a_rows, int a_cols, const __nv_bfloat16* gB,
                      int b_rows, int b_cols, Case cs, float* out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t mbar;
    __shared__ uint32_t tslot;
    uint8_t* sA = sm;
    uint8_t* sB = sm + a_rows * a_cols * 2 + 1024;
    int tid = threadIdx.x;
    // stage A and B in the chunk-major interleave layout
    for (int i = tid; i < a_rows * a_cols; i += blockDim.x) {
        int r = i / a_cols, c = i % a_cols;
        *reinterpret_cast<__nv_bfloat16*>(sA + umma::off(a_rows, r, c)) = gA[i];
    }
    for (int i = tid; i < b_rows * b_cols; i += blockDim.x) {
        int r = i / b_cols, c = i % b_cols;
        *reinterpret_cast<__nv_bfloat16*>(sB + umma::off(b_rows, r, c)) = gB[i];
    }
    if (tid == 0) {
        umma::mbar_init(&mbar, 1);
        umma::fence_mbar_init();
    }
    if (tid < 32) umma::tmem_alloc<256>(&tslot);
    umma::fence_async_smem();
    umma::fence_before_sync();
    __syncthreads();
    umma::fence_after_sync();
    uint32_t tmem = tslot;
    if (tid == 0) {
        uint32_t id = umma::idesc_bf16(128, cs.N, cs.a_mn, cs.b_mn);
        for (int k0 = 0; k0 < cs.K; k0 += 16) {
            uint64_t da, db;
            if (!cs.a_mn)  // rows = M(128), cols = K: advance 2 chunks per K step
                da = umma::desc(umma::smem_u32(sA) + (k0 / 8) * a_rows * 16, a_rows * 16, 128);
            else  // rows = K, cols = M: advance 2 row-groups per K step
                da = umma::desc(umma::smem_u32(sA) + (k0 / 8) * 128, 128, a_rows * 16);
            if (!cs.b_mn)
                db = umma::desc(umma::smem_u32(sB) + (k0 / 8) * b_rows * 16, b_rows * 16, 128);
            else
                db = umma::desc(umma::smem_u32(sB) + (k0 / 8) * 128, 128, b_rows * 16);
            umma::mma(tmem, da, db, id, k0 > 0);
        }
        umma::commit(&mbar);
    }
    umma::mbar_wait(&mbar, 0);
    umma::fence_after_sync();
    int w = tid / 32;
    for (int c0 = 0; c0 < cs.N; c0 += 16) {
        float v[16];
        umma::ld16(tmem + ((32 * w) << 16) + c0, v);
        umma::ld_wait();
        for (int j = 0; j < 16; ++j) out[tid * cs.N + c0 + j] = v[j];
    }
    umma::fence_before_sync();
    __syncthreads();
    if (tid < 32) umma::tmem_free<256>(tmem);
}

int run(Case cs, unsigned seed) {
    int M = 128;
    // A logical M x K; B logical K x N
    std::vector<float> A(M * cs.K), B(cs.K * cs.N);
    srand(seed);
    for (auto& x : A) x = float(rand() % 17 - 8) / 8.f;
    for (auto& x : B) x = float(rand() % 13 - 6) / 4.f;
    int a_rows = cs.a_mn ? cs.K : M, a_cols = cs.a_mn ? M : cs.K;
    int b_rows = cs.b_mn ? cs.K : cs.N, b_cols = cs.b_mn ? cs.N : cs.K;
    std::vector<__nv_bfloat16> hA(a_rows * a_cols), hB(b_rows * b_cols);
    for (int m = 0; m < M; ++m)
        for (int k = 0; k < cs.K; ++k)
            hA[cs.a_mn ? k * a_cols + m : m * a_cols + k] = __float2bfloat16(A[m * cs.K + k]);
    for (int k = 0; k < cs.K; ++k)
        for (int n = 0; n < cs.N; ++n)
            hB[cs.b_mn ? k * b_cols + n : n * b_cols + k] = __float2bfloat16(B[k * cs.N + n]);
    __nv_bfloat16 *dA, *dB;
    float* dO;
    cudaMalloc(&dA, hA.size() * 2);
    cudaMalloc(&dB, hB.size() * 2);
    cudaMalloc(&dO, M * cs.N * 4);
    cudaMemcpy(dA, hA.data(), hA.size() * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, hB.data(), hB.size() * 2, cudaMemcpyHostToDevice);
    size_t smem = a_rows * a_cols * 2 + 1024 + b_rows * b_cols * 2 + 1024;
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    probe<<<1, 128, smem>>>(dA, a_rows, a_cols, dB, b_rows, b_cols, cs, dO);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        printf("CUDA error %s\n", cudaGetErrorString(e));
        return 2;
    }
    std::vector<float> O(M * cs.N);
    cudaMemcpy(O.data(), dO, O.size() * 4, cudaMemcpyDeviceToHost);
    double maxerr = 0;
    for (int m = 0; m < M; ++m)
        for (int n = 0; n < cs.N; ++n) {
            double ref = 0;
            for (int k = 0; k < cs.K; ++k) ref += double(A[m * cs.K + k]) * B[k * cs.N + n];
            maxerr = fmax(maxerr, fabs(ref - O[m * cs.N + n]));
        }
    printf("N=%3d K=%3d a_mn=%d b_mn=%d  max|err|=%g  D[0][0]=%g D[127][N-1]=%g\n", cs.N, cs.K,
           cs.a_mn, cs.b_mn, maxerr, O[0], O[M * cs.N - 1]);
    cudaFree(dA);
    cudaFree(dB);
    cudaFree(dO);
    return maxerr < 1e-3 ? 0 : 1;
}

int main() {
    int bad = 0;
    Case cases[] = {{64, 16, 0, 0}, {64, 64, 0, 0}, {16, 64, 0, 0}, {48, 48, 0, 0},
                    {64, 128, 1, 1}, {16, 128, 1, 1}, {80, 128, 1, 1}, {64, 16, 0, 1},
                    {16, 64, 0, 1}, {32, 128, 1, 1}, {64, 64, 0, 1}};
    unsigned s = 1;
    for (auto& c : cases) bad += run(c, s++);
    printf(bad ? "UMMA PROBE FAILED (%d)\n" : "UMMA PROBE OK\n", bad);
    return bad ? 1 : 0;
}
