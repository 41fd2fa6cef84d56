// Microbenchmark: how fast can persistent CTAs stream a buffer through smem
// with 1-D TMA bulk copies (cp.async.bulk) and an mbarrier ring?
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void kstream(const char* src, size_t nchunks, int chunk, int nst, unsigned long long* sink) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* bar = (uint64_t*)sm; int* done = (int*)(sm + 128);
  unsigned char* st0 = sm + 256;
  int tid = threadIdx.x, lane = tid & 31;
  size_t mine = blockIdx.x < nchunks ? (nchunks - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  if (tid == 0) { for (int s = 0; s < nst; ++s) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su(&bar[s]))); done[s] = 0; }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  __syncthreads();
  auto issue = [&](size_t it, int s) {
    size_t c = blockIdx.x + it * gridDim.x;
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" :: "r"(su(&bar[s])), "r"(chunk) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      :: "r"(su(st0 + (size_t)s * chunk)), "l"(src + c * chunk), "r"(chunk), "r"(su(&bar[s])) : "memory");
  };
  if (tid == 0) for (int s = 0; s < nst && s < (int)mine; ++s) issue(s, s);
  unsigned long long acc = 0;
  for (size_t it = 0; it < mine; ++it) {
    int s = it % nst; uint32_t ph = (it / nst) & 1;
    asm volatile("{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W_%=;\n}\n" :: "r"(su(&bar[s])), "r"(ph) : "memory");
    acc += st0[(size_t)s * chunk + tid * 4];
    __syncwarp();
    if (lane == 0 && atomicAdd(&done[s], 1) == (int)blockDim.x / 32 - 1) {
      done[s] = 0;
      if (it + nst < mine) { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); issue(it + nst, s); }
    }
  }
  if (acc == 12345) *sink = acc;
}
__global__ void kread(const float4* p, size_t n, float* out) {
  float a = 0; for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) { float4 v = p[i]; a += v.x + v.w; }
  if (a == 1234.5f) *out = a;
}
int main() {
  size_t bytes = 160ull << 20; char* src; cudaMalloc(&src, bytes); cudaMemset(src, 1, bytes);
  unsigned long long* sink; cudaMalloc(&sink, 8);
  char* fl; cudaMalloc(&fl, 256 << 20);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int chunks[] = {16384, 32768}; int nsts[] = {2, 4}; int cps[] = {1, 2};
  cudaFuncSetAttribute(kstream, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int ch : chunks) for (int nst : nsts) for (int cp : cps) {
    size_t smem = 256 + (size_t)nst * ch; if (smem * cp > 227 * 1024) continue;
    size_t n = bytes / ch; float best = 1e9;
    for (int r = 0; r < 5; ++r) {
      cudaMemset(fl, r, 256 << 20); kread<<<sms * 8, 512>>>((const float4*)fl, (256 << 20) / 16, (float*)sink);
      cudaEventRecord(e0); kstream<<<sms * cp, 256, smem>>>(src, n, ch, nst, sink); cudaEventRecord(e1);
      cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    cudaError_t err = cudaGetLastError();
    printf("chunk %6d nst %d ctas/sm %d : %7.1f us  %6.0f GB/s %s\n", ch, nst, cp, best * 1e3, bytes / best / 1e6, err ? cudaGetErrorString(err) : "");
  }
  return 0;
}
