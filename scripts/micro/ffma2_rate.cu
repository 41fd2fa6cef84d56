// Microbenchmark: sustained complex multiply-accumulate rate, scalar FFMA vs packed FFMA2.
// acc[j] += conj(a) * b[j] over register-resident operands (the Gram / row-apply inner pattern).
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ u64 pk(float x, float y) { u64 r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(x), "f"(y)); return r; }
__device__ __forceinline__ float2 upk(u64 r) { float2 v; asm("mov.b64 {%0, %1}, %2;" : "=f"(v.x), "=f"(v.y) : "l"(r)); return v; }
__device__ __forceinline__ u64 fma2(u64 a, u64 b, u64 c) { u64 d; asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d; }

template <int V, int NA>
__global__ void __launch_bounds__(256) k(const float2* __restrict__ in, float2* out, int K) {
  float2 b[NA];
  for (int j = 0; j < NA; ++j) b[j] = in[threadIdx.x * NA + j];
  if (V == 0) {
    float2 acc[NA];
    for (int j = 0; j < NA; ++j) acc[j] = make_float2(0.f, 0.f);
    for (int k = 0; k < K; ++k) {
#pragma unroll
      for (int i = 0; i < NA; ++i) {
        float2 a = b[(i + 3) % NA];
#pragma unroll
        for (int j = 0; j < NA; ++j) {
          acc[j].x = fmaf(a.x, b[j].x, acc[j].x); acc[j].x = fmaf(a.y, b[j].y, acc[j].x);
          acc[j].y = fmaf(a.x, b[j].y, acc[j].y); acc[j].y = fmaf(-a.y, b[j].x, acc[j].y);
        }
      }
      b[k % NA].x += 1e-7f;
    }
    float2 s = make_float2(0.f, 0.f);
    for (int j = 0; j < NA; ++j) { s.x += acc[j].x; s.y += acc[j].y; }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  } else {
    u64 acc[NA], bb[NA];
    for (int j = 0; j < NA; ++j) { acc[j] = 0; bb[j] = pk(b[j].x, b[j].y); }
    for (int k = 0; k < K; ++k) {
#pragma unroll
      for (int i = 0; i < NA; ++i) {
        float2 a = upk(bb[(i + 3) % NA]);
        u64 ax = pk(a.x, a.x), ay = pk(a.y, -a.y);
#pragma unroll
        for (int j = 0; j < NA; ++j) {
          float2 bj = upk(bb[j]);
          acc[j] = fma2(ax, bb[j], acc[j]);
          acc[j] = fma2(ay, pk(bj.y, bj.x), acc[j]);
        }
      }
      float2 t = upk(bb[k % NA]); bb[k % NA] = pk(t.x + 1e-7f, t.y);
    }
    float2 s = make_float2(0.f, 0.f);
    for (int j = 0; j < NA; ++j) { float2 v = upk(acc[j]); s.x += v.x; s.y += v.y; }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  }
}

template <int V, int NA>
void run(int blocks_per_sm) {
  int K = 256, nb = 148 * blocks_per_sm;
  float2 *in, *out;
  cudaMalloc(&in, 256 * NA * sizeof(float2)); cudaMemset(in, 0, 256 * NA * sizeof(float2));
  cudaMalloc(&out, nb * 256 * sizeof(float2));
  k<V, NA><<<nb, 256>>>(in, out, K);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) k<V, NA><<<nb, 256>>>(in, out, K);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double cmac = 5.0 * nb * 256.0 * K * NA * NA;
  printf("V=%s NA=%d blocks/SM=%d: %.2f Tcmac/s (%.1f TFLOP/s fp32-equiv)  err=%s\n", V ? "FFMA2" : "FFMA ", NA,
         blocks_per_sm, cmac / ms / 1e9, 8 * cmac / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
  cudaFree(in); cudaFree(out);
}
int main() {
  run<0, 16>(2); run<1, 16>(2); run<0, 16>(4); run<1, 16>(4); run<0, 8>(4); run<1, 8>(4);
  return 0;
}
