// dbp_cgg.cu -- k_cgg_tc: the per-GPU sums of CG-UL's preprocessing on the tensor cores,
// G_loc = sum_{c local} H_c^H H_c and y^MRC_loc = sum_{c local} H_c^H y_c (Alg. 2 line 3 and the
// P416 footnote: the consensus of every iteration is sum_c G_c p = G_loc p), for the paths that
// keep the CG iterations separate: world > 1 (one allreduce per iteration) and
// U > 16 (UP = 32, config E) -- in place of the per-pair Grams written to HBM and summed again
// (k_prefold + k_cg_gsum).
//
// Same contraction as k_cg_tc (dbp_cgtc.cu): K = C_loc * S antenna rows per subcarrier, a CTA of
// CGG_KS warps per subcarrier, each warp streaming every CGG_KS-th stage (32 or 64 rows) through its
// own TMA ring, fp16 mma.sync m16n8k16 on an exact hi/lo split with FP32 accumulation, y^MRC on
// the FP32 cores.  Differences:
//  * UP = 32 is two 16-user halves (two 128B-swizzled boxes per stage).  The diagonal blocks use
//    the Hermitian form Z' = hi^H hi + 2 hi^H lo (G = Z' + Z'^H, two passes); the lower-left block
//    G_10 = H_1^H H_0 is formed directly, 2 G_10 ~ (2 hi_1)^H hi_0 + hi_1^H (2 lo_0) + (2 lo_1)^H hi_0
//    (three passes; lo_1^H lo_0 dropped, ~2^-22).  56 MMAs per 16 antenna rows.
//  * A running power-of-two scale per warp instead of a fresh accumulator per 32-row group: the
//    group's values are scaled by 2^-e, e = the largest exponent seen so far (warp max, redux); a
//    group with a larger maximum rescales the accumulator by the exact factor 2^(2 (e_old - e_new))
//    first.  Values below the running maximum keep an absolute error <= 2^-24 of it.
//  * The result goes to HBM: G_loc [N][tri(UP)] packed lower triangle, y^MRC [N][UP] (J = 1).
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "dbp_device.cuh"
#include "dbp_internal.h"
#include "dbp_tc.cuh"

namespace dbp {

constexpr int CGG_KS = 2, CGG_NST = 2;

struct CggArgs {
    int N, C, S, U, S16, CB, R, nstages, pitch;   // pitch: bytes per ring stage
    float2* G;            // [N][tri(UP)]
    float2* mrc;          // [N][UP]
};

template <int UP>
struct CGG {
    static constexpr int UH = UP / 16;                       // 16-user halves
    static constexpr int NT = UH == 1 ? 4 : 12;              // accumulator tiles (m16 x n8)
    static constexpr int NMF = 4 * UH;                       // y^MRC partial floats per lane (x2: a, b)
    static constexpr int XW = NT * 4 + 2 * NMF;              // exchange floats per lane
    static constexpr int TRI = UP * (UP + 1) / 2;
    __host__ __device__ static size_t warp_bytes(int pitch) { return (size_t)CGG_NST * pitch + 1024; }
    // ring (+ mbarriers in the 1024-B tail) per warp; after the stream a warp's partials go to its own
    // ring, and warp 0's ring holds Z [UP][UP+1] + y^MRC [UP]
    static size_t smem(int pitch) { return 1024 + CGG_KS * warp_bytes(pitch); }
};

__device__ __forceinline__ unsigned h2x(unsigned a) {          // 2 a, exact in fp16
    unsigned r;
    asm("add.rn.f16x2 %0, %1, %1;" : "=r"(r) : "r"(a));
    return r;
}

// T += A^H B over one K16 step for one m16 x n16 complex block: T[0], T[1] Re (columns 0-7, 8-15),
// T[2], T[3] Im; A, B fragments (Re, Im) in the f = uh + 2 kh order of dbp_tc.cuh.
__device__ __forceinline__ void cgg_blk(float (*T)[4], const unsigned (&ar)[4], const unsigned (&ai)[4],
                                        const unsigned (&br)[4], const unsigned (&bi)[4]) {
    mma_f16(T[0], ar[0], ar[1], ar[2], ar[3], br[0], br[2]);
    mma_f16(T[1], ar[0], ar[1], ar[2], ar[3], br[1], br[3]);
    mma_f16(T[2], ar[0], ar[1], ar[2], ar[3], bi[0], bi[2]);
    mma_f16(T[3], ar[0], ar[1], ar[2], ar[3], bi[1], bi[3]);
    mma_f16(T[0], ai[0], ai[1], ai[2], ai[3], bi[0], bi[2]);
    mma_f16(T[1], ai[0], ai[1], ai[2], ai[3], bi[1], bi[3]);
    mma_f16(T[2], ai[0], ai[1], ai[2], ai[3], br[0] ^ TC_NEG2, br[2] ^ TC_NEG2);
    mma_f16(T[3], ai[0], ai[1], ai[2], ai[3], br[1] ^ TC_NEG2, br[3] ^ TC_NEG2);
}

// fp16 fragments of one K16 step of one half, values scaled by sc: hi, 2 lo
__device__ __forceinline__ void cgg_frag(const float2 (&v)[2][2][2], float sc, unsigned (&rh)[4], unsigned (&ih)[4],
                                         unsigned (&rl)[4], unsigned (&il)[4]) {
#pragma unroll
    for (int f = 0; f < 4; ++f) {
        const int uh = f & 1, kh = f >> 1;
        float2 h2[2], l2[2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const float2 xs = __fmul2_rn(v[uh][kh][e], make_float2(sc, sc));
            h2[e] = make_float2(__uint_as_float(__float_as_uint(xs.x) & 0xffffe000u),
                                __uint_as_float(__float_as_uint(xs.y) & 0xffffe000u));
            l2[e] = __ffma2_rn(h2[e], make_float2(-1.f, -1.f), xs);                  // exact
        }
        rh[f] = f16x2(h2[0].x, h2[1].x);
        ih[f] = f16x2(h2[0].y, h2[1].y);
        rl[f] = h2x(f16x2(l2[0].x, l2[1].x));
        il[f] = h2x(f16x2(l2[0].y, l2[1].y));
    }
}

template <int UP>
__global__ void __launch_bounds__(CGG_KS * 32)
k_cgg_tc(const __grid_constant__ CUtensorMap tmH, const __grid_constant__ CUtensorMap tmY, CggArgs a) {
    using Q = CGG<UP>;
    constexpr int UH = Q::UH, NT = Q::NT, TRI = Q::TRI;
    constexpr int GK = 2 / UH;                              // K16 steps per scale group (32 values per lane)
    extern __shared__ __align__(128) unsigned char smem_raw[];
    DBP_POISON_SMEM(smem_raw);
    griddep_launch();
    unsigned char* const base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, t4 = lane & 3;
    const int R = a.R, pitch = a.pitch;
    unsigned char* const ring = base + (size_t)warp * Q::warp_bytes(pitch);           // 1024-aligned stages
    uint64_t* const bar = reinterpret_cast<uint64_t*>(ring + (size_t)CGG_NST * pitch);
    float2* const zs = reinterpret_cast<float2*>(base);                               // [UP][UP + 1], warp 0's ring
    float2* const ms = zs + UP * (UP + 1);                                             // [UP]
    // a ring holds >= CGG_NST stages of >= UH * 4096 + 1024 bytes (32 rows of UH halves, y, 1024-B pitch)
    static_assert((UP * (UP + 1) + UP) * 8 <= CGG_NST * (UH * 4096 + 1024) &&
                  Q::XW * 32 * 4 <= CGG_NST * (UH * 4096 + 1024), "hand-off fits a ring");
    const int n = blockIdx.x;
    const int nmine = (a.nstages - warp + CGG_KS - 1) / CGG_KS;

    auto issue = [&](int j) {                               // the warp's j-th stage: H halves, then y
        const int sl = j % CGG_NST, c0 = (warp + j * CGG_KS) * a.CB;
        unsigned char* dst = ring + (size_t)sl * pitch;
        mbar_arrive_expect_tx(&bar[sl], (uint32_t)(R * (128 * UH + 8)));
#pragma unroll
        for (int h = 0; h < UH; ++h) tma_load4(dst + h * R * 128, &tmH, 16 * h, 0, n, c0, &bar[sl]);
        tma_load4(dst + UH * R * 128, &tmY, 0, 0, n, c0, &bar[sl]);
    };
    if (lane == 0) {
        for (int s = 0; s < CGG_NST; ++s) mbar_init(&bar[s], 1);
        fence_mbar_init();
        for (int j = 0; j < CGG_NST && j < nmine; ++j) issue(j);
    }
    DBP_SYNCWARP();

    float T[NT][4];
#pragma unroll
    for (int i = 0; i < NT; ++i)
#pragma unroll
        for (int e = 0; e < 4; ++e) T[i][e] = 0.f;
    float2 mfa[UH][2], mfb[UH][2];
#pragma unroll
    for (int h = 0; h < UH; ++h)
#pragma unroll
        for (int uh = 0; uh < 2; ++uh) mfa[h][uh] = mfb[h][uh] = make_float2(0.f, 0.f);
    int erun = -126;                                        // running exponent (T is in units of 2^(2 erun - 1))

    for (int i = 0; i < nmine; ++i) {
        const int sl = i % CGG_NST;
        mbar_wait(&bar[sl], (uint32_t)((i / CGG_NST) & 1));
        const unsigned char* stage = ring + (size_t)sl * pitch;
        const float2* yv = reinterpret_cast<const float2*>(stage + UH * R * 128);
        for (int kq = 0; kq < R / (16 * GK); ++kq) {        // scale groups of GK K16 steps
            float2 v[GK][UH][2][2][2];                      // [K16 step][half][uh][kh][e]
#pragma unroll
            for (int k = 0; k < GK; ++k)
#pragma unroll
                for (int h = 0; h < UH; ++h) tc16_load<false>(v[k][h], stage + h * R * 128, GK * kq + k, g, t4);
            float mx = 0.f;
#pragma unroll
            for (int k = 0; k < GK; ++k)
#pragma unroll
                for (int h = 0; h < UH; ++h)
#pragma unroll
                    for (int q8 = 0; q8 < 8; ++q8) {
                        const float2 x = v[k][h][q8 >> 2][(q8 >> 1) & 1][q8 & 1];
                        mx = fmaxf(mx, fmaxf(fabsf(x.x), fabsf(x.y)));
                    }
            unsigned mxb;
            asm volatile("redux.sync.max.u32 %0, %1, 0xffffffff;" : "=r"(mxb) : "r"(__float_as_uint(mx)));
            const int eg = mxb ? (int)((mxb >> 23) & 0xff) - 127 : -126;
            if (eg > erun) {                                // warp-uniform: rescale to the new maximum
                const float f = __int_as_float(max(1, 127 + 2 * (erun - eg)) << 23);   // 2^(2 (erun - eg)), >= 2^-126
#pragma unroll
                for (int t = 0; t < NT; ++t)
#pragma unroll
                    for (int e = 0; e < 4; ++e) T[t][e] *= f;
                erun = eg;
            }
            const float sc = __int_as_float((127 - erun) << 23);
            // y^MRC, FP32, unscaled: mfa += (hr, hi) (yr, yi), mfb += (hr, hi) (yi, yr)
#pragma unroll
            for (int k = 0; k < GK; ++k)
#pragma unroll
                for (int kh = 0; kh < 2; ++kh) {
                    const float4 yy =
                        *reinterpret_cast<const float4*>(yv + 16 * (GK * kq + k) + 8 * kh + 2 * t4);
                    const float2 y0 = make_float2(yy.x, yy.y), y1 = make_float2(yy.z, yy.w);
                    const float2 s0 = make_float2(yy.y, yy.x), s1 = make_float2(yy.w, yy.z);
#pragma unroll
                    for (int h = 0; h < UH; ++h)
#pragma unroll
                        for (int uh = 0; uh < 2; ++uh) {
                            mfa[h][uh] = __ffma2_rn(v[k][h][uh][kh][0], y0, mfa[h][uh]);
                            mfb[h][uh] = __ffma2_rn(v[k][h][uh][kh][0], s0, mfb[h][uh]);
                            mfa[h][uh] = __ffma2_rn(v[k][h][uh][kh][1], y1, mfa[h][uh]);
                            mfb[h][uh] = __ffma2_rn(v[k][h][uh][kh][1], s1, mfb[h][uh]);
                        }
                }
#pragma unroll
            for (int k = 0; k < GK; ++k) {
                unsigned rh0[4], ih0[4], rl0[4], il0[4];
                cgg_frag(v[k][0], sc, rh0, ih0, rl0, il0);
                cgg_blk(&T[0], rh0, ih0, rh0, ih0);         // Z'_00 = hi^H hi + 2 hi^H lo
                cgg_blk(&T[0], rh0, ih0, rl0, il0);
                if constexpr (UH == 2) {
                    unsigned rh1[4], ih1[4], rl1[4], il1[4];
                    cgg_frag(v[k][1], sc, rh1, ih1, rl1, il1);
                    cgg_blk(&T[4], rh1, ih1, rh1, ih1);     // Z'_11
                    cgg_blk(&T[4], rh1, ih1, rl1, il1);
                    unsigned rh2[4], ih2[4];
#pragma unroll
                    for (int f = 0; f < 4; ++f) { rh2[f] = h2x(rh1[f]); ih2[f] = h2x(ih1[f]); }
                    cgg_blk(&T[8], rh2, ih2, rh0, ih0);     // 2 G_10: (2 hi_1)^H hi_0
                    cgg_blk(&T[8], rh1, ih1, rl0, il0);     //        + hi_1^H (2 lo_0)
                    cgg_blk(&T[8], rl1, il1, rh0, ih0);     //        + (2 lo_1)^H hi_0
                }
            }
        }
        DBP_SYNCWARP();                                     // every lane's reads of the slot are done
        if (lane == 0 && i + CGG_NST < nmine) {
            fence_proxy_async();
            issue(i + CGG_NST);
        }
    }

    // to true units (exact power of two), then warps 1.. hand their partials to warp 0 (fixed order)
#pragma unroll
    for (int t = 0; t < NT; ++t)
#pragma unroll
        for (int e = 0; e < 4; ++e) T[t][e] = ldexpf(T[t][e], 2 * erun - 1);
    float mr[UH][2][2];                                     // H^H y partial (Re, Im) per (half, uh)
#pragma unroll
    for (int h = 0; h < UH; ++h)
#pragma unroll
        for (int uh = 0; uh < 2; ++uh) {
            mr[h][uh][0] = mfa[h][uh].x + mfa[h][uh].y;
            mr[h][uh][1] = mfb[h][uh].x - mfb[h][uh].y;
        }
    if (warp > 0) {
        float* xw = reinterpret_cast<float*>(ring);                         // the warp's own (drained) ring
#pragma unroll
        for (int q = 0; q < NT * 4; ++q) xw[q * 32 + lane] = T[q >> 2][q & 3];
#pragma unroll
        for (int q = 0; q < 4 * UH; ++q) xw[(NT * 4 + q) * 32 + lane] = mr[q >> 2][(q >> 1) & 1][q & 1];
    }
    DBP_SYNCTHREADS();
    if (warp == 0) {
        DBP_SYNCWARP();
        for (int w = 1; w < CGG_KS; ++w) {
            const float* xw = reinterpret_cast<const float*>(base + (size_t)w * Q::warp_bytes(pitch));
#pragma unroll
            for (int q = 0; q < NT * 4; ++q) T[q >> 2][q & 3] += xw[q * 32 + lane];
#pragma unroll
            for (int q = 0; q < 4 * UH; ++q) mr[q >> 2][(q >> 1) & 1][q & 1] += xw[(NT * 4 + q) * 32 + lane];
        }
        // tiles -> Z [UP][UP + 1]: block (rh, ch) tile element e at row 16 rh + g + 8 (e >> 1),
        // column 16 ch + 8 nb + 2 t + (e & 1); blocks 00, 11 (Z'), 10 (G_10)
#pragma unroll
        for (int b = 0; b < NT / 4; ++b) {
            const int r0 = b == 0 ? 0 : 16, c0 = b == 1 ? 16 : 0;
#pragma unroll
            for (int nb = 0; nb < 2; ++nb)
#pragma unroll
                for (int e = 0; e < 4; ++e)
                    zs[(r0 + g + 8 * (e >> 1)) * (UP + 1) + c0 + 8 * nb + 2 * t4 + (e & 1)] =
                        make_float2(T[4 * b + nb][e], T[4 * b + 2 + nb][e]);
        }
#pragma unroll
        for (int h = 0; h < UH; ++h)
#pragma unroll
            for (int uh = 0; uh < 2; ++uh) {
                float2 m = make_float2(mr[h][uh][0], mr[h][uh][1]);
#pragma unroll
                for (int o = 1; o < 4; o <<= 1) {
                    m.x += __shfl_xor_sync(0xffffffffu, m.x, o);
                    m.y += __shfl_xor_sync(0xffffffffu, m.y, o);
                }
                if (t4 == 0) ms[16 * h + 8 * uh + g] = m;
            }
    }
    DBP_SYNCTHREADS();
    griddep_wait();
    float2* Gn = a.G + (size_t)n * TRI;
    for (int e = threadIdx.x; e < TRI; e += blockDim.x) {
        int r = (int)((sqrtf(8.f * (float)e + 1.f) - 1.f) * 0.5f);
        while ((r + 1) * (r + 2) / 2 <= e) ++r;
        while (r * (r + 1) / 2 > e) --r;
        const int c = e - r * (r + 1) / 2;
        float2 v = zs[r * (UP + 1) + c];
        if ((r >> 4) == (c >> 4)) {                         // diagonal block: G = Z' + Z'^H
            const float2 zt = zs[c * (UP + 1) + r];
            v = make_float2(v.x + zt.x, r == c ? 0.f : v.y - zt.y);
        }
        Gn[e] = v;
    }
    if (threadIdx.x < UP) a.mrc[(size_t)n * UP + threadIdx.x] = ms[threadIdx.x];
}

bool cgg_tc_ok(int UP, int J, int N, int C, int S, int U) {
    return (UP == 16 || UP == 32) && J == 1 && N > 0 && C > 0 && S > 0 && S <= 64 && U % 2 == 0;
}

// G_loc and y^MRC_loc of the rank's clusters (cgg_tc_ok shapes); false: not taken
bool launch_cgg_tc(const LaunchCtx& L, int UP, const float2* H, const float2* y, int C, int N, int S, int U,
                   float2* G, float2* mrc) {
    if (!cgg_tc_ok(UP, 1, N, C, S, U)) return false;
    CggArgs a{};
    a.N = N; a.C = C; a.S = S; a.U = U; a.G = G; a.mrc = mrc;
    a.S16 = S <= 16 ? 16 : (S + 31) / 32 * 32;
    a.R = std::max(32, a.S16);
    a.CB = a.R / a.S16;
    a.nstages = (C + a.CB - 1) / a.CB;
    a.pitch = ((UP / 16) * a.R * 128 + a.R * 8 + 1023) / 1024 * 1024;
    CUtensorMap tmH{}, tmY{};
    if (!make_map4(&tmH, H, U, S, N, C, 16, a.S16, 1, a.CB, true)) return false;
    if (!make_map4(&tmY, y, S, 1, N, C, a.S16, 1, 1, a.CB)) return false;
    const size_t smem = UP == 16 ? CGG<16>::smem(a.pitch) : CGG<32>::smem(a.pitch);
    auto k = UP == 16 ? k_cgg_tc<16> : k_cgg_tc<32>;
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    if (!launch_pdl(k, N, CGG_KS * 32, smem, L, tmH, tmY, a)) return false;
    L.count(1);
    return true;
}

}  // namespace dbp
