// Microbenchmark: streaming 157 MB (config C's H) through per-warp 1-D bulk-copy rings of small
// chunks (k_cg_tc's shape: 4 KB per stage), as a function of chunk size, ring depth and warps per
// SM, in two orders: contiguous (warp w takes chunks w, w + W, ...) and k_cg_tc's (one subcarrier
// n per warp, its C = 32 cluster blocks 4.9 MB apart).  Plus an LDG.128 grid-stride read.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/micro/tma_small scripts/micro/tma_small.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// one warp = one ring of nst stages of `chunk` bytes; warp gw streams items gw, gw + nw, ...; an item
// is `per` chunks: chunk j of item i at byte offset off(i, j)
__global__ void kwarp(const char* src, int nitems, int per, int chunk, int nst, int strided, size_t stride,
                      unsigned long long* sink) {
    extern __shared__ __align__(1024) unsigned char sm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, wpc = blockDim.x >> 5;
    unsigned char* ring = sm + (size_t)warp * (nst * chunk + 1024);
    uint64_t* bar = (uint64_t*)(ring + (size_t)nst * chunk);
    const int gw = blockIdx.x * wpc + warp, nw = gridDim.x * wpc;
    const int myitems = gw < nitems ? (nitems - 1 - gw) / nw + 1 : 0;
    const long total = (long)myitems * per;
    auto off = [&](long q) {
        const long it = q / per, j = q % per;
        const long item = gw + it * nw;
        return strided ? (size_t)j * stride + (size_t)item * chunk : ((size_t)item * per + j) * chunk;
    };
    auto issue = [&](long q) {
        const int s = q % nst;
        asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bar[s])), "r"(chunk)
                     : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         su(ring + (size_t)s * chunk)),
                     "l"(src + off(q)), "r"(chunk), "r"(su(&bar[s]))
                     : "memory");
    };
    if (lane == 0) {
        for (int s = 0; s < nst; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar[s])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int s = 0; s < nst && s < total; ++s) issue(s);
    }
    __syncwarp();
    unsigned long long acc = 0;
    for (long q = 0; q < total; ++q) {
        const int s = q % nst;
        const uint32_t ph = (q / nst) & 1;
        asm volatile("{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W_%=;\n}\n" ::"r"(
                         su(&bar[s])),
                     "r"(ph)
                     : "memory");
        acc += ring[(size_t)s * chunk + lane * 4];
        __syncwarp();
        if (lane == 0 && q + nst < total) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue(q + nst);
        }
    }
    if (acc == 12345) *sink = acc;
}

__global__ void kread(const float4* p, size_t n, float* out) {
    float a = 0;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        float4 v = p[i];
        a += v.x + v.w;
    }
    if (a == 1234.5f) *out = a;
}

int main() {
    const int C = 32, N = 1200;
    const size_t bytes = (size_t)C * N * 4096;
    char* src;
    cudaMalloc(&src, bytes);
    cudaMemset(src, 1, bytes);
    unsigned long long* sink;
    cudaMalloc(&sink, 8);
    char* fl;
    cudaMalloc(&fl, 256 << 20);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaFuncSetAttribute(kwarp, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto flush = [&](int r) {
        cudaMemset(fl, r, 256 << 20);
        kread<<<sms * 8, 512>>>((const float4*)fl, (256 << 20) / 16, (float*)sink);
    };
    {
        float best = 1e9;
        for (int r = 0; r < 5; ++r) {
            flush(r);
            cudaEventRecord(e0);
            kread<<<sms * 8, 512>>>((const float4*)src, bytes / 16, (float*)sink);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (ms < best) best = ms;
        }
        printf("LDG.128 grid-stride: %7.1f us %6.0f GB/s\n", best * 1e3, bytes / best / 1e6);
    }
    const int chunks[] = {4096, 8192, 16384};
    const int nsts[] = {2, 3, 4, 6};
    const int wpcs[] = {2, 4};
    for (int strided = 0; strided < 2; ++strided)
        for (int ch : chunks)
            for (int nst : nsts)
                for (int wpc : wpcs) {
                    const size_t per_warp = (size_t)nst * ch + 1024;
                    const size_t smem = per_warp * wpc;
                    if (smem > 227 * 1024) continue;
                    int occ = 0;
                    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kwarp, wpc * 32, smem);
                    // item = one subcarrier (C chunks of 4 KB = C * 4096 / ch chunks of ch bytes)
                    const int per = C * 4096 / ch;
                    const int nitems = N;
                    const int grid = (nitems + wpc - 1) / wpc;
                    float best = 1e9;
                    for (int r = 0; r < 5; ++r) {
                        flush(r);
                        cudaEventRecord(e0);
                        kwarp<<<grid, wpc * 32, smem>>>(src, nitems, per, ch, nst, strided, (size_t)N * ch, sink);
                        cudaEventRecord(e1);
                        cudaEventSynchronize(e1);
                        float ms;
                        cudaEventElapsedTime(&ms, e0, e1);
                        if (ms < best) best = ms;
                    }
                    cudaError_t err = cudaGetLastError();
                    printf("%s chunk %5d nst %d warps/cta %d (%2d warps/SM): %7.1f us %6.0f GB/s %s\n",
                           strided ? "strided " : "contig  ", ch, nst, wpc, occ * wpc, best * 1e3, bytes / best / 1e6,
                           err ? cudaGetErrorString(err) : "");
                }
    return 0;
}
