// Microbenchmark: the folded-row UL Gram inner loop (dbp_fold.cuh fold_gram_ul) on
// shared-memory data with no TMA, 3 CTAs x 4 warps per SM as in k_fused.  Reports the
// complex-MAC rate so the fused kernel's Gram phase can be compared with its ceiling.
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_1702_04458_b200/csrc/dbp_fold.cuh"
using namespace dbp;
constexpr int UP = 16;
using F = Fold<UP>;
using G = FoldStage<UP, false, true>;

__global__ void __launch_bounds__(128, 3) kgram(float2* out, int iters) {
    extern __shared__ __align__(128) unsigned char sm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float2* stage = reinterpret_cast<float2*>(sm) + warp * (G::STG / 8);
    for (int e = lane; e < G::HSZ + G::YSZ; e += 32) stage[e] = make_float2(1e-3f * e, -2e-3f * e);
    __syncwarp();
    const int q = lane / F::L, l = lane % F::L;
    int row[4];
    for (int m = 0; m < 4; ++m) row[m] = F::row(m, l);
    f2x A[F::NSLOT], E[4];
    for (int e = 0; e < F::NSLOT; ++e) A[e] = 0ull;
    for (int m = 0; m < 4; ++m) E[m] = 0ull;
    for (int i = 0; i < iters; ++i) fold_gram_ul<UP, true>(A, E, stage, q, row);
    float2 acc = make_float2(0.f, 0.f);
    for (int e = 0; e < F::NSLOT; ++e) acc = c_add(acc, upk2(A[e]));
    for (int m = 0; m < 4; ++m) acc = c_add(acc, upk2(E[m]));
    out[blockIdx.x * 128 + threadIdx.x] = acc;
}

int main() {
    int blocks = 148 * 3, iters = 2000;
    size_t smem = 4 * G::STG;
    float2* out;
    cudaMalloc(&out, blocks * 128 * sizeof(float2));
    cudaFuncSetAttribute(kgram, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kgram<<<blocks, 128, smem>>>(out, 10);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    kgram<<<blocks, 128, smem>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    // per stage per lane: 40 slots + 4 MF = 44 cmac x SC antennas
    double cmac = (double)blocks * 128 * iters * F::SC * (F::NSLOT + 4);
    printf("gram loop: %.2f Tcmac/s (%.1f TFLOP/s, %.0f%% of 74.4)  %s\n", cmac / ms / 1e9, 8 * cmac / ms / 1e9,
           100 * 8 * cmac / ms / 1e9 / 74.4, cudaGetErrorString(cudaGetLastError()));
    return 0;
}
