// Microbenchmark: is the per-pair Hermitian Gram H_c^H H_c
// (P295; S = 32 antennas, U = 16 users, config C) faster on the legacy warp-level
// tensor path (mma.sync m16n8k8 TF32, split into hi + lo for ~fp32 accuracy)
// than on FP32 FFMA2 (the folded-row loop: 6.16 T complex MAC/s measured)?
//
//  1. peak rates of register-only mma.sync loops: tf32 m16n8k8, f16/bf16 m16n8k16;
//  2. the Gram itself from HBM: one pair per warp (M = 16 users, N = 32 = [Re G | Im G],
//     K = 64 = [Re h; Im h] per antenna), the H fragments loaded straight from global
//     memory (each lane's 16 complex values are 128 B; the warp reads the pair's 4 KB
//     exactly once, every 256-B warp load fully used), one pair prefetched ahead;
//     passes = 1 (plain TF32), 2 (hi*hi + hi*lo + lo*hi folded as hi*(hi+lo) + lo*hi
//     ... see below) or 3 (hi*hi + hi*lo + lo*hi).  Reports pairs/s, the useful
//     complex-MAC rate (S * U(U+1)/2 per pair) and the error against an fp64 Gram.
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

__device__ __forceinline__ unsigned tf32(float x) {
    unsigned r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ void mma_tf32(float (&d)[4], const unsigned (&a)[4], unsigned b0, unsigned b1) {
    asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                 : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
                 : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void mma_f16(float (&d)[4], const unsigned (&a)[4], unsigned b0, unsigned b1) {
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                 : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
                 : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void mma_bf16(float (&d)[4], const unsigned (&a)[4], unsigned b0, unsigned b1) {
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                 : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
                 : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

template <int KIND>
__global__ void k_peak(float* out, int iters) {
    unsigned a[4];
    for (int i = 0; i < 4; ++i) a[i] = 0x3c003c00u + threadIdx.x + i;
    float d[8][4] = {};
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            if (KIND == 0) mma_tf32(d[j], a, a[j & 3], a[(j + 1) & 3]);
            else if (KIND == 1) mma_f16(d[j], a, a[j & 3], a[(j + 1) & 3]);
            else mma_bf16(d[j], a, a[j & 3], a[(j + 1) & 3]);
        }
    }
    float s = 0.f;
    for (int j = 0; j < 8; ++j) s += d[j][0] + d[j][1] + d[j][2] + d[j][3];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// One pair per warp iteration.  Lane (g = lane/4, t = lane%4) holds h[i] = H[s_i][u_i] for
// s in {8kk + t, 8kk + t + 4} (kk = 0..3), u in {g, g + 8}: the A fragment (rows u,
// K = antenna re|im) and -- since B's Re columns are A^T -- every B fragment too.
template <int PASSES>
__global__ void __launch_bounds__(128) k_gram(const float2* __restrict__ H, float* __restrict__ Gout, int P) {
    const int lane = threadIdx.x & 31;
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    const int g = lane >> 2, t = lane & 3;
    float2 h[16], hn[16];
    auto load = [&](float2 (&dst)[16], int p) {
        const float2* Hp = H + (size_t)p * 512;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int s = 8 * kk + t + ((e >> 1) << 2), u = g + ((e & 1) << 3);
                dst[kk * 4 + e] = __ldcs(Hp + s * 16 + u);
            }
    };
    int p = gw;
    if (p < P) load(h, p);
    for (; p < P; p += nw) {
        if (p + nw < P) load(hn, p + nw);
        float acc[4][4] = {};     // n-tiles: Re cols 0-7, Re 8-15, Im 0-7, Im 8-15
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
            // A fragments (rows u = g, g+8; k = t, t+4): re part (k-step kk), im part (k-step kk+4)
            unsigned rh[4], ih[4], rl[4], il[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                // fragment order a0 (g, t), a1 (g+8, t), a2 (g, t+4), a3 (g+8, t+4)
                const int src = kk * 4 + ((e & 1) ? 1 : 0) + ((e & 2) ? 2 : 0);
                const float2 v = h[src];
                rh[e] = tf32(v.x);
                ih[e] = tf32(v.y);
                rl[e] = tf32(v.x - __uint_as_float(rh[e]));
                il[e] = tf32(v.y - __uint_as_float(ih[e]));
            }
            // Re G: sum_k Hr_u Hr_n + Hi_u Hi_n;  Im G: sum_k Hr_u Hi_n - Hi_u Hr_n
            // B fragment for Re tile n0 (cols 0-7) = {a0, a2}, tile n1 (cols 8-15) = {a1, a3}
            auto pass = [&](const unsigned (&ar)[4], const unsigned (&ai)[4], const unsigned (&br)[4],
                            const unsigned (&bi)[4]) {
                mma_tf32(acc[0], ar, br[0], br[2]);
                mma_tf32(acc[0], ai, bi[0], bi[2]);
                mma_tf32(acc[1], ar, br[1], br[3]);
                mma_tf32(acc[1], ai, bi[1], bi[3]);
                mma_tf32(acc[2], ar, bi[0], bi[2]);
                mma_tf32(acc[2], ai, br[0] ^ 0x80000000u, br[2] ^ 0x80000000u);
                mma_tf32(acc[3], ar, bi[1], bi[3]);
                mma_tf32(acc[3], ai, br[1] ^ 0x80000000u, br[3] ^ 0x80000000u);
            };
            pass(rh, ih, rh, ih);
            if (PASSES >= 2) pass(rh, ih, rl, il);
            if (PASSES >= 3) pass(rl, il, rh, ih);
        }
        // D fragment: c0 (g, 2t), c1 (g, 2t+1), c2 (g+8, 2t), c3 (g+8, 2t+1) per n-tile
        float* Gp = Gout + (size_t)p * 512;          // [16][16] re, then [16][16] im
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) {
            const int col = (nt & 1) * 8 + 2 * t, off = (nt >> 1) * 256;
            *reinterpret_cast<float2*>(Gp + off + g * 16 + col) = make_float2(acc[nt][0], acc[nt][1]);
            *reinterpret_cast<float2*>(Gp + off + (g + 8) * 16 + col) = make_float2(acc[nt][2], acc[nt][3]);
        }
#pragma unroll
        for (int i = 0; i < 16; ++i) h[i] = hn[i];
    }
}


// f16 m16n8k16 variant: per-pair power-of-two pre-scale (warp max |re|, |im| -> [1, 2)) so
// hi = fp16(a), lo = fp16(a - hi) stay normal over 2^-13 .. 2 of the pair's largest entry;
// G is un-scaled exactly.  Lane (g, t) holds, per K16 step kk, H[16kk + {2t, 2t+1, 2t+8, 2t+9}][{g, g+8}].
#include <cuda_fp16.h>
__device__ __forceinline__ unsigned h2u(__half2 v) { return *reinterpret_cast<unsigned*>(&v); }
template <int PASSES, bool STORE>
__global__ void __launch_bounds__(128) k_gram16(const float2* __restrict__ H, float* __restrict__ Gout, int P) {
    const int lane = threadIdx.x & 31;
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    const int g = lane >> 2, t = lane & 3;
    float2 h[16], hn[16];
    // index i = kk * 8 + kp * 4 + ub * 2 + ko: k = 16kk + 2t + 8kp + ko, u = g + 8ub
    auto load = [&](float2 (&dst)[16], int p) {
        const float2* Hp = H + (size_t)p * 512;
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            const int kk = i >> 3, kp = (i >> 2) & 1, ub = (i >> 1) & 1, ko = i & 1;
            dst[i] = __ldcs(Hp + (16 * kk + 2 * t + 8 * kp + ko) * 16 + g + 8 * ub);
        }
    };
    int p = gw;
    if (p < P) load(h, p);
    float checksum = 0.f;
    for (; p < P; p += nw) {
        if (p + nw < P) load(hn, p + nw);
        float mx = 0.f;
#pragma unroll
        for (int i = 0; i < 16; ++i) mx = fmaxf(mx, fmaxf(fabsf(h[i].x), fabsf(h[i].y)));
#pragma unroll
        for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        const int ex = mx > 0.f ? ((__float_as_int(mx) >> 23) & 0xff) - 127 : 0;
        const float sc = __int_as_float((127 - ex) << 23);          // 2^-ex
        float acc[4][4] = {};
#pragma unroll
        for (int kk = 0; kk < 2; ++kk) {
            // A regs: r0 = {A[g][2t], A[g][2t+1]}, r1 = {A[g+8][..]}, r2 = {A[g][2t+8], ..}, r3 = {A[g+8][2t+8], ..}
            unsigned rh[4], ih[4], rl[4], il[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int ub = e & 1, kp = e >> 1;
                const float2 v0 = h[kk * 8 + kp * 4 + ub * 2], v1 = h[kk * 8 + kp * 4 + ub * 2 + 1];
                const float a0 = v0.x * sc, a1 = v1.x * sc, b0 = v0.y * sc, b1 = v1.y * sc;
                const __half2 hr = __floats2half2_rn(a0, a1), hi = __floats2half2_rn(b0, b1);
                rh[e] = h2u(hr);
                ih[e] = h2u(hi);
                rl[e] = h2u(__floats2half2_rn(a0 - __low2float(hr), a1 - __high2float(hr)));
                il[e] = h2u(__floats2half2_rn(b0 - __low2float(hi), b1 - __high2float(hi)));
            }
            auto pass = [&](const unsigned (&ar)[4], const unsigned (&ai)[4], const unsigned (&br)[4],
                            const unsigned (&bi)[4]) {
                mma_f16(acc[0], ar, br[0], br[2]);
                mma_f16(acc[0], ai, bi[0], bi[2]);
                mma_f16(acc[1], ar, br[1], br[3]);
                mma_f16(acc[1], ai, bi[1], bi[3]);
                mma_f16(acc[2], ar, bi[0], bi[2]);
                mma_f16(acc[2], ai, br[0] ^ 0x80008000u, br[2] ^ 0x80008000u);
                mma_f16(acc[3], ar, bi[1], bi[3]);
                mma_f16(acc[3], ai, br[1] ^ 0x80008000u, br[3] ^ 0x80008000u);
            };
            pass(rh, ih, rh, ih);
            if (PASSES >= 3) {
                pass(rh, ih, rl, il);
                pass(rl, il, rh, ih);
            }
        }
        const float us = __int_as_float((127 + 2 * ex) << 23);     // 2^(2 ex)
        if (STORE) {
            float* Gp = Gout + (size_t)p * 512;
#pragma unroll
            for (int nt = 0; nt < 4; ++nt) {
                const int col = (nt & 1) * 8 + 2 * t, off = (nt >> 1) * 256;
                *reinterpret_cast<float2*>(Gp + off + g * 16 + col) = make_float2(acc[nt][0] * us, acc[nt][1] * us);
                *reinterpret_cast<float2*>(Gp + off + (g + 8) * 16 + col) = make_float2(acc[nt][2] * us, acc[nt][3] * us);
            }
        } else {
#pragma unroll
            for (int nt = 0; nt < 4; ++nt) checksum += (acc[nt][0] + acc[nt][1] + acc[nt][2] + acc[nt][3]) * us;
        }
#pragma unroll
        for (int i = 0; i < 16; ++i) h[i] = hn[i];
    }
    if (!STORE && checksum == 12345.f) Gout[0] = checksum;
}

int main(int argc, char** argv) {
    int dev = 0, sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    float* out;
    CK(cudaMalloc(&out, (size_t)sms * 8 * 256 * 4));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const char* names[3] = {"tf32 m16n8k8", "f16 m16n8k16", "bf16 m16n8k16"};
    for (int kind = 0; kind < 3; ++kind) {
        const int iters = 4000;
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(e0);
            if (kind == 0) k_peak<0><<<sms * 8, 256>>>(out, iters);
            if (kind == 1) k_peak<1><<<sms * 8, 256>>>(out, iters);
            if (kind == 2) k_peak<2><<<sms * 8, 256>>>(out, iters);
            cudaEventRecord(e1);
            CK(cudaEventSynchronize(e1));
        }
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double flop_per = kind == 0 ? 16.0 * 8 * 8 * 2 : 16.0 * 8 * 16 * 2;
        const double flops = (double)sms * 8 * 8 * iters * 8 * flop_per;   // warps x iters x 8 mma
        printf("peak %-14s %8.1f TFLOP/s\n", names[kind], flops / ms / 1e9);
    }

    const int P = 38400;                     // config C: 32 clusters x 1200 subcarriers
    std::vector<float2> h((size_t)P * 512);
    srand(1);
    for (auto& v : h) v = make_float2((rand() / (float)RAND_MAX - 0.5f) * 2.f, (rand() / (float)RAND_MAX - 0.5f) * 2.f);
    float2* dH;
    float* dG;
    CK(cudaMalloc(&dH, h.size() * 8));
    CK(cudaMalloc(&dG, (size_t)P * 512 * 4));
    CK(cudaMemcpy(dH, h.data(), h.size() * 8, cudaMemcpyHostToDevice));
    void* flush;
    CK(cudaMalloc(&flush, 256 << 20));
    std::vector<float> G((size_t)P * 512);
    auto check = [&](float us, const char* name) {
        CK(cudaMemcpy(G.data(), dG, G.size() * 4, cudaMemcpyDeviceToHost));
        double err = 0, nrm = 0;
        for (int p = 0; p < P; p += 97) {
            const float2* hp = h.data() + (size_t)p * 512;
            for (int u = 0; u < 16; ++u)
                for (int n = 0; n < 16; ++n) {
                    double re = 0, im = 0;
                    for (int s = 0; s < 32; ++s) {
                        const float2 a = hp[s * 16 + u], b = hp[s * 16 + n];
                        re += (double)a.x * b.x + (double)a.y * b.y;
                        im += (double)a.x * b.y - (double)a.y * b.x;
                    }
                    const double dr = G[(size_t)p * 512 + u * 16 + n] - re;
                    const double di = G[(size_t)p * 512 + 256 + u * 16 + n] - im;
                    err += dr * dr + di * di;
                    nrm += re * re + im * im;
                }
        }
        const double cmac = (double)P * 32 * 136;
        printf("%-28s %7.1f us  %.2f T useful cmac/s  HBM %.0f GB/s  rel err %.2e\n", name, us, cmac / us / 1e6,
               (double)P * (4096 + 2048) / us / 1e3, std::sqrt(err / nrm));
    };
    auto timeit = [&](auto launch) {
        float best = 1e9;
        for (int rep = 0; rep < 6; ++rep) {
            cudaMemset(flush, rep, 256 << 20);
            cudaEventRecord(e0);
            launch();
            cudaEventRecord(e1);
            CK(cudaEventSynchronize(e1));
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (rep) best = std::min(best, ms);
        }
        return best * 1e3f;
    };
    char nm[64];
    for (int cpb : {4, 8, 12}) {
        const int grid = sms * cpb;
        cudaMemset(dG, 0, (size_t)P * 512 * 4);
        float us = timeit([&] { k_gram<3><<<grid, 128>>>(dH, dG, P); });
        snprintf(nm, sizeof nm, "tf32x3 store, %d CTA/SM", cpb); check(us, nm);
        us = timeit([&] { k_gram16<1, true><<<grid, 128>>>(dH, dG, P); });
        snprintf(nm, sizeof nm, "f16x1 store, %d CTA/SM", cpb); check(us, nm);
        us = timeit([&] { k_gram16<3, true><<<grid, 128>>>(dH, dG, P); });
        snprintf(nm, sizeof nm, "f16x3 store, %d CTA/SM", cpb); check(us, nm);
        us = timeit([&] { k_gram16<3, false><<<grid, 128>>>(dH, dG, P); });
        printf("f16x3 no store, %2d CTA/SM    %7.1f us\n", cpb, us);
    }
    // scale robustness: the same H times 2^-20 and 2^+20 (path loss / large gains)
    for (float f : {9.5367431640625e-07f, 1048576.f}) {
        std::vector<float2> hs(h);
        for (auto& v : hs) { v.x *= f; v.y *= f; }
        CK(cudaMemcpy(dH, hs.data(), hs.size() * 8, cudaMemcpyHostToDevice));
        k_gram16<3, true><<<sms * 8, 128>>>(dH, dG, P);
        CK(cudaDeviceSynchronize());
        CK(cudaMemcpy(G.data(), dG, G.size() * 4, cudaMemcpyDeviceToHost));
        for (auto& v : G) v /= (double)f * f;
        CK(cudaMemcpy(dG, G.data(), G.size() * 4, cudaMemcpyHostToDevice));
        snprintf(nm, sizeof nm, "f16x3 H scaled by %g", f); check(0.f, nm);
    }
    return 0;
}
