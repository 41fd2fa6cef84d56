// dbp_cgtc.cu -- k_cg_tc: decentralized CG-UL (Alg. 2) at world == 1 with the cluster-summed Gram on
// the tensor cores.
//
// CG never needs a cluster's own Gram: the consensus of its preprocessing and every iteration is a
// sum over clusters, G = sum_c H_c^H H_c (P416 footnote) and y^MRC = sum_c H_c^H y_c (line 3), i.e.
// one Gram with K = C * S antennas per subcarrier (1024 at configs B-D scale).  Unlike the per-pair
// Grams of ADMM (K = 32, dbp_tc.cuh: measured slower than FP32 there), this long-K contraction is
// what the tensor cores are for.  KS warps (2, or 1 for short K) own one subcarrier: each warp streams
// every KS-th stage of the subcarrier's clusters through its own TMA ring (R = 32 or 64 antenna rows x
// 16 users per stage, 128B swizzle), each 32-row group runs mma.sync m16n8k16 FP16 in dbp_tc.cuh's
// split form (below), y^MRC runs on the FP32 cores from the same registers; the warps' partial sums
// meet in shared memory (fixed order), and warp 0 runs the T CG iterations on the assembled G
// (replicated update, shuffle dot products, P404-409, P715).  The warps synchronise once, at the
// end; 1200 subcarriers x 2 warps fit one wave at 10 CTAs per SM.  (43.7 us at
// config C against a measured ~32-36 us floor for streaming the 157 MB through such rings.)
//
// Split (exact to ~2^-22 relative): per 32-row group the warp scales its values by an exact power
// of two (max |Re|, |Im| -> [1, 2)), v = hi + lo with hi = v truncated to fp16's 11 bits; then
// Z' = hi^H hi + 2 hi^H lo (A = hi, B = hi then B = 2 lo: two MMA passes) is added to the running
// FP32 sum with the exact factor 2^(2 e - 1), and G = Z' + Z'^H (the 1/2 inside the factor), which
// is hi^H hi + hi^H lo + lo^H hi = G - lo^H lo.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "dbp_device.cuh"
#include "dbp_internal.h"
#include "dbp_lanerow.cuh"
#include "dbp_tc.cuh"

namespace dbp {

constexpr int CGT_WARPS = 2, CGT_NST = 2;   // warps per CTA, ring stages per warp

struct CgTcArgs {
    int N, C, S, U, T, S16, CB, R, nstages;
    float rho;
    Modem md;
    float2* x_hat;        // [N][U]
    uint8_t* hard;        // [N][U] or null
};

// per warp: H ring [NST][R][128 B] | y ring [NST][R] float2 | mbarriers [NST], 1024-B pitch
__host__ __device__ inline size_t cgtc_warp_bytes(int R) {
    const size_t b = (size_t)CGT_NST * R * 128 + (size_t)CGT_NST * R * 8 + CGT_NST * 8;
    return (b + 1023) / 1024 * 1024;
}
// k_cg_tcj: the y ring holds J symbols per row; after the stream the lead ring also holds y^MRC [8][16]
// and four CG lines
__host__ __device__ inline size_t cgtcj_warp_bytes(int R, int J) {
    const size_t b = (size_t)CGT_NST * R * 128 + (size_t)CGT_NST * R * J * 8 + CGT_NST * 8;
    return (b + 1023) / 1024 * 1024;
}
static size_t cgtc_smem(int R) {
    // the hand-off (a warp's partials: its own drained ring; Z' scratch + CG line: the subcarrier's
    // first warp's ring) needs no memory of its own: 10 CTAs (20 warps) per SM
    return 1024 + CGT_WARPS * cgtc_warp_bytes(R);
}

__device__ __forceinline__ unsigned hadd2u(unsigned a, unsigned b) {
    unsigned r;
    asm("add.rn.f16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
    return r;
}

// One 32-row group (two K16 steps) of the stage: Z' += 2^(2e-1) (hi^H hi + 2 hi^H lo), mf += H^H y.
__device__ __forceinline__ void cgtc_group(float (&acc)[4][4], float2 (&mfa)[2], float2 (&mfb)[2], const unsigned char* stage,
                                           const float2* yv, int kk0, int g, int t4) {
    float2 v[2][2][2][2];                                   // [K16 step][uh][kh][e]
    tc16_load<false>(v[0], stage, kk0, g, t4);
    tc16_load<false>(v[1], stage, kk0 + 1, g, t4);
    float m4[4];                                            // tree max (short dependency chains)
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        m4[q] = 0.f;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const float2 x = v[q >> 1][q & 1][e >> 1][e & 1];
            m4[q] = fmaxf(m4[q], fmaxf(fabsf(x.x), fabsf(x.y)));
        }
    }
    const float mx = fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3]));
    // non-negative floats order as their bit patterns: one integer max-reduction for the warp
    unsigned mxb;
    asm volatile("redux.sync.max.u32 %0, %1, 0xffffffff;" : "=r"(mxb) : "r"(__float_as_uint(mx)));
    const int ex = mxb ? (int)((mxb >> 23) & 0xff) - 127 : 0;
    const float sc = __int_as_float((127 - ex) << 23);      // 2^-e: max -> [1, 2)
    // y^MRC on the FP32 cores, unscaled, packed: mfa += (hr, hi) (yr, yi), mfb += (hr, hi) (yi, yr), so
    // conj(h) y = (mfa.x + mfa.y) + i (mfb.x - mfb.y) at the end
#pragma unroll
    for (int k = 0; k < 2; ++k)
#pragma unroll
        for (int kh = 0; kh < 2; ++kh) {
            const float4 yy = *reinterpret_cast<const float4*>(yv + 16 * (kk0 + k) + 8 * kh + 2 * t4);
            const float2 y0 = make_float2(yy.x, yy.y), y1 = make_float2(yy.z, yy.w);
            const float2 s0 = make_float2(yy.y, yy.x), s1 = make_float2(yy.w, yy.z);
#pragma unroll
            for (int uh = 0; uh < 2; ++uh) {
                mfa[uh] = __ffma2_rn(v[k][uh][kh][0], y0, mfa[uh]);
                mfb[uh] = __ffma2_rn(v[k][uh][kh][0], s0, mfb[uh]);
                mfa[uh] = __ffma2_rn(v[k][uh][kh][1], y1, mfa[uh]);
                mfb[uh] = __ffma2_rn(v[k][uh][kh][1], s1, mfb[uh]);
            }
        }
    float st[4][4];
#pragma unroll
    for (int q4 = 0; q4 < 4; ++q4)
#pragma unroll
        for (int e = 0; e < 4; ++e) st[q4][e] = 0.f;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        // fragments: f = uh + 2 kh (a0: uh 0 kh 0, a1: uh 1 kh 0, a2: uh 0 kh 1, a3: uh 1 kh 1)
        unsigned rh[4], ih[4], rl[4], il[4];
#pragma unroll
        for (int f = 0; f < 4; ++f) {
            const int uh = f & 1, kh = f >> 1;
            float2 h2[2], l2[2];                            // (re, im) pairs: packed FP32x2 ops
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const float2 xs = __fmul2_rn(v[k][uh][kh][e], make_float2(sc, sc));
                h2[e] = make_float2(__uint_as_float(__float_as_uint(xs.x) & 0xffffe000u),
                                    __uint_as_float(__float_as_uint(xs.y) & 0xffffe000u));
                l2[e] = __ffma2_rn(h2[e], make_float2(-1.f, -1.f), xs);     // exact
            }
            rh[f] = f16x2(h2[0].x, h2[1].x);
            ih[f] = f16x2(h2[0].y, h2[1].y);
            rl[f] = f16x2(l2[0].x, l2[1].x);
            il[f] = f16x2(l2[0].y, l2[1].y);
            rl[f] = hadd2u(rl[f], rl[f]);                   // 2 lo, exact in fp16
            il[f] = hadd2u(il[f], il[f]);
        }
        // Re tiles A_re B_re + A_im B_im, Im tiles A_re B_im - A_im B_re (dbp_tc.cuh tc16_gram_pair);
        // consecutive MMAs go to different tiles (a dependent MMA is four issues back)
#pragma unroll
        for (int pass = 0; pass < 2; ++pass) {
            const unsigned* Br = pass ? rl : rh;
            const unsigned* Bi = pass ? il : ih;
            mma_f16(st[0], rh[0], rh[1], rh[2], rh[3], Br[0], Br[2]);
            mma_f16(st[1], rh[0], rh[1], rh[2], rh[3], Br[1], Br[3]);
            mma_f16(st[2], rh[0], rh[1], rh[2], rh[3], Bi[0], Bi[2]);
            mma_f16(st[3], rh[0], rh[1], rh[2], rh[3], Bi[1], Bi[3]);
            mma_f16(st[0], ih[0], ih[1], ih[2], ih[3], Bi[0], Bi[2]);
            mma_f16(st[1], ih[0], ih[1], ih[2], ih[3], Bi[1], Bi[3]);
            mma_f16(st[2], ih[0], ih[1], ih[2], ih[3], Br[0] ^ TC_NEG2, Br[2] ^ TC_NEG2);
            mma_f16(st[3], ih[0], ih[1], ih[2], ih[3], Br[1] ^ TC_NEG2, Br[3] ^ TC_NEG2);
        }
    }
    // 2^(2e - 1): an exponent field when it has one (|h| between 2^-62 and 2^64), else ldexpf (0 / inf /
    // subnormal -- where the Gram itself leaves the FP32 range)
    const int e2 = 2 * ex - 1;
    const float us = (e2 >= -126 && e2 <= 127) ? __int_as_float((127 + e2) << 23) : ldexpf(1.f, e2);
#pragma unroll
    for (int q4 = 0; q4 < 4; ++q4)
#pragma unroll
        for (int e = 0; e < 4; ++e) acc[q4][e] = fmaf(st[q4][e], us, acc[q4][e]);
}

// KS warps per subcarrier (K split; 2 at configs C / D, 1 when a subcarrier has few stages, e.g.
// config B: no hand-off, and the CTA's two warps solve two subcarriers independently)
template <int KS>
__global__ void __launch_bounds__(CGT_WARPS * 32, 9)
k_cg_tc(const __grid_constant__ CUtensorMap tmH, const __grid_constant__ CUtensorMap tmY, CgTcArgs a) {
    constexpr int UP = 16, SPC = CGT_WARPS / KS;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    DBP_POISON_SMEM(smem_raw);
    griddep_launch();
    unsigned char* const base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, t4 = lane & 3;
    const int R = a.R;
    unsigned char* const ring = base + (size_t)warp * cgtc_warp_bytes(R);   // 1024-aligned stages
    float2* const yring = reinterpret_cast<float2*>(ring + (size_t)CGT_NST * R * 128);
    uint64_t* const bar = reinterpret_cast<uint64_t*>(yring + (size_t)CGT_NST * R);
    const int wk = warp % KS;                               // the warp's share of its subcarrier's stages
    unsigned char* const lead = base + (size_t)(warp - wk) * cgtc_warp_bytes(R);   // the subcarrier's first warp
    float2* const zs = reinterpret_cast<float2*>(lead);    // its ring, after the stream
    float2* const P = zs + 16 * 17;
    static_assert((16 * 17 + 16) * 8 <= CGT_NST * 32 * 128 && 20 * 32 * 4 <= CGT_NST * 32 * 128, "hand-off fits");
    const int n = blockIdx.x * SPC + warp / KS;
    if (n >= a.N) return;                                   // KS = 1 only (warp-uniform; no CTA barrier then)
    const int nmine = (a.nstages - wk + KS - 1) / KS;      // this warp: stages wk, wk + KS, ..

    auto issue = [&](int j) {                               // the warp's j-th stage
        const int sl = j % CGT_NST, c0 = (wk + j * KS) * a.CB;
        mbar_arrive_expect_tx(&bar[sl], (uint32_t)(R * (128 + 8)));
        tma_load4(ring + (size_t)sl * R * 128, &tmH, 0, 0, n, c0, &bar[sl]);
        tma_load4(yring + (size_t)sl * R, &tmY, 0, 0, n, c0, &bar[sl]);
    };
    if (lane == 0) {
        for (int s = 0; s < CGT_NST; ++s) mbar_init(&bar[s], 1);
        fence_mbar_init();
        for (int j = 0; j < CGT_NST && j < nmine; ++j) issue(j);
    }
    DBP_SYNCWARP();

    float acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int e = 0; e < 4; ++e) acc[i][e] = 0.f;
    float2 mfa[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)}, mfb[2] = {mfa[0], mfa[0]};
    for (int i = 0; i < nmine; ++i) {
        const int sl = i % CGT_NST;
        mbar_wait(&bar[sl], (uint32_t)((i / CGT_NST) & 1));
        const unsigned char* stage = ring + (size_t)sl * R * 128;
        const float2* yv = yring + (size_t)sl * R;
#ifndef DBP_EXP_CGTC_NOCOMP
#define DBP_EXP_CGTC_NOCOMP 0   // experiment only: stream the stages without the Gram (wrong results)
#endif
        if (!DBP_EXP_CGTC_NOCOMP)
            for (int gq = 0; gq < R / 32; ++gq) cgtc_group(acc, mfa, mfb, stage, yv, 2 * gq, g, t4);
        DBP_SYNCWARP();                                     // every lane's reads of the slot are done
        if (lane == 0 && i + CGT_NST < nmine) {
            fence_proxy_async();
            issue(i + CGT_NST);
        }
    }

    // warps 1.. of the subcarrier hand their partials to its first warp, which adds them in warp order
    if constexpr (KS > 1) {
        if (wk > 0) {
            float* xw = reinterpret_cast<float*>(ring);  // the warp's own drained ring
#pragma unroll
            for (int q = 0; q < 16; ++q) xw[q * 32 + lane] = acc[q >> 2][q & 3];
#pragma unroll
            for (int uh = 0; uh < 2; ++uh) {
                xw[(16 + 2 * uh) * 32 + lane] = mfa[uh].x + mfa[uh].y;
                xw[(17 + 2 * uh) * 32 + lane] = mfb[uh].x - mfb[uh].y;
            }
        }
        DBP_SYNCTHREADS();
        if (wk > 0) return;
    }
    for (int w = 1; w < KS; ++w) {
        const float* xw = reinterpret_cast<const float*>(lead + (size_t)w * cgtc_warp_bytes(R));
#pragma unroll
        for (int q = 0; q < 16; ++q) acc[q >> 2][q & 3] += xw[q * 32 + lane];
#pragma unroll
        for (int uh = 0; uh < 2; ++uh) {
            mfa[uh].x += xw[(16 + 2 * uh) * 32 + lane];     // (mfa.y, mfb.y): folded below
            mfb[uh].x += xw[(17 + 2 * uh) * 32 + lane];
        }
    }
    // G = Z' + Z'^H through the scratch; y^MRC summed over each quad's 4 lanes
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int e1 = 0; e1 < 2; ++e1)
#pragma unroll
            for (int cc = 0; cc < 2; ++cc)
                zs[(g + 8 * e1) * 17 + 8 * h + 2 * t4 + cc] = make_float2(acc[h][2 * e1 + cc], acc[2 + h][2 * e1 + cc]);
#pragma unroll
    for (int uh = 0; uh < 2; ++uh) {
        float2 m = make_float2(mfa[uh].x + mfa[uh].y, mfb[uh].x - mfb[uh].y);
#pragma unroll
        for (int o = 1; o < 4; o <<= 1) {
            m.x += __shfl_xor_sync(0xffffffffu, m.x, o);
            m.y += __shfl_xor_sync(0xffffffffu, m.y, o);
        }
        if (t4 == 0) P[g + 8 * uh] = m;
    }
    DBP_SYNCWARP();
    // lines 6-18: r = y^MRC, p = r, x = 0; T iterations (rho = N0/Es, reading 10); 16 lanes per CG,
    // the upper half-warp a duplicate (full-mask shuffles)
    const int u = lane % UP;
    float2 grow[UP];
#pragma unroll
    for (int jc = 0; jc < UP; ++jc) {
        const float2 z = zs[u * 17 + jc], zt = zs[jc * 17 + u];
        grow[jc] = make_float2(z.x + zt.x, z.y - zt.y);
    }
    float2 r = P[u], p = r, x = make_float2(0.f, 0.f);
    float rr = group_sum<UP>(c_norm2(r));
    for (int t = 0; t < a.T; ++t) {
        DBP_SYNCWARP();
        if (lane < UP) P[u] = p;
        DBP_SYNCWARP();
        float2 pv[UP];
        read_vec<UP>(P, pv);
        float2 w4[4] = {};                                  // four partial sums: short FMA chains
#pragma unroll
        for (int jc = 0; jc < UP; ++jc) c_fma(w4[jc & 3], grow[jc], pv[jc]);
        const float2 w = c_add(c_add(w4[0], w4[1]), c_add(w4[2], w4[3]));
        cg_update<UP>(x, r, p, rr, w, a.rho);
    }
    griddep_wait();
    if (lane < UP && u < a.U) {
        a.x_hat[(size_t)n * a.U + u] = x;
        if (a.hard) a.hard[(size_t)n * a.U + u] = slice_bits(x, a.md);
    }
}

// ----------------------------------------------------------------------------------------------
// k_cg_tcj: N_sym = J in 2..8 (the coherence block of P706-709; Table II: J = 7).  The subcarrier's
// Gram is formed once (as above) and serves all J symbols.  The J matched filters H^H y_j go to the
// tensor cores too (FP32 cores would need 8 J accumulator registers per lane): B = [y_0 .. y_J-1]
// as one n8 tile (lane (g, t) holds symbol g), 2 MF ~ hi^H (2 y_hi) + hi^H (2 y_lo) + (2 lo)^H y_hi
// (three passes, 12 MMAs per K16 step; y scaled by its own power of two).  A running exponent per
// warp (dbp_cgg.cu) replaces the per-group fresh accumulators, for both H and y, so the kernel stays
// at <= 112 registers (one wave of 1200 CTAs).  The J CG solves run on half-warps, two per warp.
struct CgTcjArgs {
    CgTcArgs b;
    int J;
};

__device__ __forceinline__ float p2f(int e) {           // 2^e, exact, any int e (0 / inf beyond FP32)
    return (e >= -126 && e <= 127) ? __int_as_float((127 + e) << 23) : ldexpf(1.f, e);
}

template <int KS>
__global__ void __maxnreg__(112)   // no spills, 9 CTAs (18 warps) per SM: 1200 subcarriers in one wave
k_cg_tcj(const __grid_constant__ CUtensorMap tmH, const __grid_constant__ CUtensorMap tmY, CgTcjArgs aj) {
    constexpr int UP = 16, SPC = CGT_WARPS / KS;
    const CgTcArgs& a = aj.b;
    const int J = aj.J;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    DBP_POISON_SMEM(smem_raw);
    griddep_launch();
    unsigned char* const base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, t4 = lane & 3;
    const int R = a.R, S16 = a.S16;
    const size_t wb = cgtcj_warp_bytes(R, J);
    unsigned char* const ring = base + (size_t)warp * wb;
    float2* const yring = reinterpret_cast<float2*>(ring + (size_t)CGT_NST * R * 128);
    uint64_t* const bar = reinterpret_cast<uint64_t*>(yring + (size_t)CGT_NST * R * J);
    const int wk = warp % KS;
    unsigned char* const lead = base + (size_t)(warp - wk) * wb;
    float2* const zs = reinterpret_cast<float2*>(lead);    // [16][17], then y^MRC [8][16], CG lines [4][16]
    float2* const mrc = zs + 16 * 17;
    float2* const P = mrc + 8 * UP;
    const int n = blockIdx.x * SPC + warp / KS;
    if (n >= a.N) return;                                   // KS = 1 only (warp-uniform)
    const int nmine = (a.nstages - wk + KS - 1) / KS;

    auto issue = [&](int j) {
        const int sl = j % CGT_NST, c0 = (wk + j * KS) * a.CB;
        mbar_arrive_expect_tx(&bar[sl], (uint32_t)(R * (128 + 8 * J)));
        tma_load4(ring + (size_t)sl * R * 128, &tmH, 0, 0, n, c0, &bar[sl]);
        tma_load4(yring + (size_t)sl * R * J, &tmY, 0, 0, n, c0, &bar[sl]);
    };
    if (lane == 0) {
        for (int s2 = 0; s2 < CGT_NST; ++s2) mbar_init(&bar[s2], 1);
        fence_mbar_init();
        for (int j = 0; j < CGT_NST && j < nmine; ++j) issue(j);
    }
    DBP_SYNCWARP();

    float acc[4][4], mf[2][4];                              // Z' tiles; 2 MF tiles (Re, Im): users x symbols
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int e = 0; e < 4; ++e) acc[i][e] = 0.f;
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int e = 0; e < 4; ++e) mf[i][e] = 0.f;
    int eh = -126, ey = -126;                               // running exponents of H and y
    const bool gy = g < J;                                  // this lane's symbol column exists
    for (int i = 0; i < nmine; ++i) {
        const int sl = i % CGT_NST;
        mbar_wait(&bar[sl], (uint32_t)((i / CGT_NST) & 1));
        const unsigned char* stage = ring + (size_t)sl * R * 128;
        const float2* yst = yring + (size_t)sl * R * J;     // [CB][J][S16]
        for (int gq = 0; gq < R / 32; ++gq) {
            float2 v[2][2][2][2];                           // H: [K16 step][uh][kh][e]
            float2 yv[2][2][2];                             // y of symbol g: [K16 step][kh][e]
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                const int kk = 2 * gq + k;
                tc16_load<false>(v[k], stage, kk, g, t4);
                const int r0 = 16 * kk, cb = r0 / S16, s0 = r0 - cb * S16;
#pragma unroll
                for (int kh = 0; kh < 2; ++kh) {
                    float4 q = make_float4(0.f, 0.f, 0.f, 0.f);
                    if (gy) q = *reinterpret_cast<const float4*>(yst + ((size_t)cb * J + g) * S16 + s0 + 8 * kh + 2 * t4);
                    yv[k][kh][0] = make_float2(q.x, q.y);
                    yv[k][kh][1] = make_float2(q.z, q.w);
                }
            }
            float mh = 0.f, my = 0.f;
#pragma unroll
            for (int k = 0; k < 2; ++k)
#pragma unroll
                for (int q8 = 0; q8 < 8; ++q8) {
                    const float2 x = v[k][q8 >> 2][(q8 >> 1) & 1][q8 & 1];
                    mh = fmaxf(mh, fmaxf(fabsf(x.x), fabsf(x.y)));
                }
#pragma unroll
            for (int k = 0; k < 2; ++k)
#pragma unroll
                for (int q4 = 0; q4 < 4; ++q4) {
                    const float2 x = yv[k][q4 >> 1][q4 & 1];
                    my = fmaxf(my, fmaxf(fabsf(x.x), fabsf(x.y)));
                }
            unsigned mhb, myb;
            asm volatile("redux.sync.max.u32 %0, %1, 0xffffffff;" : "=r"(mhb) : "r"(__float_as_uint(mh)));
            asm volatile("redux.sync.max.u32 %0, %1, 0xffffffff;" : "=r"(myb) : "r"(__float_as_uint(my)));
            const int gh = mhb ? (int)((mhb >> 23) & 0xff) - 127 : -126;
            const int gyx = myb ? (int)((myb >> 23) & 0xff) - 127 : -126;
            if (gh > eh || gyx > ey) {                      // warp-uniform: rescale to the new maxima
                const int dh = max(gh - eh, 0), dy = max(gyx - ey, 0);
                const float fz = p2f(-2 * dh), fm = p2f(-dh - dy);
#pragma unroll
                for (int t = 0; t < 4; ++t)
#pragma unroll
                    for (int e = 0; e < 4; ++e) acc[t][e] *= fz;
#pragma unroll
                for (int t = 0; t < 2; ++t)
#pragma unroll
                    for (int e = 0; e < 4; ++e) mf[t][e] *= fm;
                eh += dh;
                ey += dy;
            }
            const float sh = p2f(-eh), sy = p2f(-ey);
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                unsigned rh[4], ih[4], rl[4], il[4];
#pragma unroll
                for (int f = 0; f < 4; ++f) {
                    const int uh = f & 1, kh = f >> 1;
                    float2 h2[2], l2[2];
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const float2 xs = __fmul2_rn(v[k][uh][kh][e], make_float2(sh, sh));
                        h2[e] = make_float2(__uint_as_float(__float_as_uint(xs.x) & 0xffffe000u),
                                            __uint_as_float(__float_as_uint(xs.y) & 0xffffe000u));
                        l2[e] = __ffma2_rn(h2[e], make_float2(-1.f, -1.f), xs);
                    }
                    rh[f] = f16x2(h2[0].x, h2[1].x);
                    ih[f] = f16x2(h2[0].y, h2[1].y);
                    rl[f] = hadd2u(f16x2(l2[0].x, l2[1].x), f16x2(l2[0].x, l2[1].x));    // 2 lo
                    il[f] = hadd2u(f16x2(l2[0].y, l2[1].y), f16x2(l2[0].y, l2[1].y));
                }
                // y of symbol g: B fragments b0 (kh = 0), b1 (kh = 1); yh = hi, Y2 = 2 hi, L2 = 2 lo
                unsigned yhr[2], yhi[2], y2r[2], y2i[2], l2r[2], l2i[2];
#pragma unroll
                for (int kh = 0; kh < 2; ++kh) {
                    float2 h2[2], l2[2];
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const float2 xs = __fmul2_rn(yv[k][kh][e], make_float2(sy, sy));
                        h2[e] = make_float2(__uint_as_float(__float_as_uint(xs.x) & 0xffffe000u),
                                            __uint_as_float(__float_as_uint(xs.y) & 0xffffe000u));
                        l2[e] = __ffma2_rn(h2[e], make_float2(-1.f, -1.f), xs);
                    }
                    yhr[kh] = f16x2(h2[0].x, h2[1].x);
                    yhi[kh] = f16x2(h2[0].y, h2[1].y);
                    y2r[kh] = hadd2u(yhr[kh], yhr[kh]);
                    y2i[kh] = hadd2u(yhi[kh], yhi[kh]);
                    const unsigned lr = f16x2(l2[0].x, l2[1].x), li = f16x2(l2[0].y, l2[1].y);
                    l2r[kh] = hadd2u(lr, lr);
                    l2i[kh] = hadd2u(li, li);
                }
                // Gram: Z' = hi^H hi + 2 hi^H lo (tiles as in cgtc_group)
#pragma unroll
                for (int pass = 0; pass < 2; ++pass) {
                    const unsigned* Br = pass ? rl : rh;
                    const unsigned* Bi = pass ? il : ih;
                    mma_f16(acc[0], rh[0], rh[1], rh[2], rh[3], Br[0], Br[2]);
                    mma_f16(acc[1], rh[0], rh[1], rh[2], rh[3], Br[1], Br[3]);
                    mma_f16(acc[2], rh[0], rh[1], rh[2], rh[3], Bi[0], Bi[2]);
                    mma_f16(acc[3], rh[0], rh[1], rh[2], rh[3], Bi[1], Bi[3]);
                    mma_f16(acc[0], ih[0], ih[1], ih[2], ih[3], Bi[0], Bi[2]);
                    mma_f16(acc[1], ih[0], ih[1], ih[2], ih[3], Bi[1], Bi[3]);
                    mma_f16(acc[2], ih[0], ih[1], ih[2], ih[3], Br[0] ^ TC_NEG2, Br[2] ^ TC_NEG2);
                    mma_f16(acc[3], ih[0], ih[1], ih[2], ih[3], Br[1] ^ TC_NEG2, Br[3] ^ TC_NEG2);
                }
                // 2 MF: A = hi with B = 2 y_hi and B = 2 y_lo, then A = 2 lo with B = y_hi
                mma_f16(mf[0], rh[0], rh[1], rh[2], rh[3], y2r[0], y2r[1]);
                mma_f16(mf[1], rh[0], rh[1], rh[2], rh[3], y2i[0], y2i[1]);
                mma_f16(mf[0], ih[0], ih[1], ih[2], ih[3], y2i[0], y2i[1]);
                mma_f16(mf[1], ih[0], ih[1], ih[2], ih[3], y2r[0] ^ TC_NEG2, y2r[1] ^ TC_NEG2);
                mma_f16(mf[0], rh[0], rh[1], rh[2], rh[3], l2r[0], l2r[1]);
                mma_f16(mf[1], rh[0], rh[1], rh[2], rh[3], l2i[0], l2i[1]);
                mma_f16(mf[0], ih[0], ih[1], ih[2], ih[3], l2i[0], l2i[1]);
                mma_f16(mf[1], ih[0], ih[1], ih[2], ih[3], l2r[0] ^ TC_NEG2, l2r[1] ^ TC_NEG2);
                mma_f16(mf[0], rl[0], rl[1], rl[2], rl[3], yhr[0], yhr[1]);
                mma_f16(mf[1], rl[0], rl[1], rl[2], rl[3], yhi[0], yhi[1]);
                mma_f16(mf[0], il[0], il[1], il[2], il[3], yhi[0], yhi[1]);
                mma_f16(mf[1], il[0], il[1], il[2], il[3], yhr[0] ^ TC_NEG2, yhr[1] ^ TC_NEG2);
            }
        }
        DBP_SYNCWARP();
        if (lane == 0 && i + CGT_NST < nmine) {
            fence_proxy_async();
            issue(i + CGT_NST);
        }
    }
    // to true units: G = 2^(2 eh - 1) (Z' + Z'^H), MF = 2^(eh + ey - 1) MF'
    const float fg = p2f(2 * eh - 1), fmf = p2f(eh + ey - 1);
#pragma unroll
    for (int t = 0; t < 4; ++t)
#pragma unroll
        for (int e = 0; e < 4; ++e) acc[t][e] *= fg;
#pragma unroll
    for (int t = 0; t < 2; ++t)
#pragma unroll
        for (int e = 0; e < 4; ++e) mf[t][e] *= fmf;
    if constexpr (KS > 1) {
        if (wk > 0) {
            float* xw = reinterpret_cast<float*>(ring);  // the warp's own drained ring
#pragma unroll
            for (int q = 0; q < 16; ++q) xw[q * 32 + lane] = acc[q >> 2][q & 3];
#pragma unroll
            for (int q = 0; q < 8; ++q) xw[(16 + q) * 32 + lane] = mf[q >> 2][q & 3];
        }
        DBP_SYNCTHREADS();
        if (wk == 0) {
            for (int w = 1; w < KS; ++w) {
                const float* xw = reinterpret_cast<const float*>(lead + (size_t)w * wb);
#pragma unroll
                for (int q = 0; q < 16; ++q) acc[q >> 2][q & 3] += xw[q * 32 + lane];
#pragma unroll
                for (int q = 0; q < 8; ++q) mf[q >> 2][q & 3] += xw[(16 + q) * 32 + lane];
            }
        }
        DBP_SYNCTHREADS();                                  // the other rings are read: zs may overwrite
    }
    if (wk == 0) {
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int e1 = 0; e1 < 2; ++e1)
#pragma unroll
                for (int cc = 0; cc < 2; ++cc)
                    zs[(g + 8 * e1) * 17 + 8 * h + 2 * t4 + cc] =
                        make_float2(acc[h][2 * e1 + cc], acc[2 + h][2 * e1 + cc]);
        // MF tile element e: user g + 8 (e >> 1), symbol 2 t + (e & 1)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const int jj = 2 * t4 + (e & 1);
            mrc[jj * UP + g + 8 * (e >> 1)] = make_float2(mf[0][e], mf[1][e]);
        }
    }
    if constexpr (KS > 1) DBP_SYNCTHREADS();
    else DBP_SYNCWARP();
    // the J CG solves (lines 6-18) on half-warps: system jb = 2 (warp's index in the subcarrier) + half + 2 KS r
    const int u = lane % UP, half = lane / UP;
    float2 grow[UP];
#pragma unroll
    for (int jc = 0; jc < UP; ++jc) {
        const float2 z = zs[u * 17 + jc], zt = zs[jc * 17 + u];
        grow[jc] = make_float2(z.x + zt.x, z.y - zt.y);
    }
    float2* Pl = P + (2 * wk + half) * UP;
    const int rounds = (J + 2 * KS - 1) / (2 * KS);        // warp-uniform trip count
    for (int rr0 = 0; rr0 < rounds; ++rr0) {
        const int jb = 2 * wk + half + 2 * KS * rr0;
        const bool live = jb < J;
        float2 r = live ? mrc[jb * UP + u] : make_float2(0.f, 0.f), p = r, x = make_float2(0.f, 0.f);
        float rr = group_sum<UP>(c_norm2(r));
        for (int t = 0; t < a.T; ++t) {
            DBP_SYNCWARP();
            Pl[u] = p;
            DBP_SYNCWARP();
            float2 pv[UP];
            read_vec<UP>(Pl, pv);
            float2 w4[4] = {};
#pragma unroll
            for (int jc = 0; jc < UP; ++jc) c_fma(w4[jc & 3], grow[jc], pv[jc]);
            const float2 w = c_add(c_add(w4[0], w4[1]), c_add(w4[2], w4[3]));
            cg_update<UP>(x, r, p, rr, w, a.rho);
        }
        griddep_wait();
        if (live && u < a.U) {
            const size_t o = ((size_t)n * J + jb) * a.U + u;
            a.x_hat[o] = x;
            if (a.hard) a.hard[o] = slice_bits(x, a.md);
        }
    }
}

bool cg_tc_ok(int UP, int J, int N, int C, int S) {
    return UP == 16 && J >= 1 && J <= 8 && N > 0 && C > 0 && S > 0 && S <= 64;
}

// CG-UL at world 1, N_sym <= 8, 9 <= U <= 16 (UP = 16), S <= 64: one kernel (false: not taken)
bool launch_cg_tc(const LaunchCtx& L, int UP, const float2* H, const float2* y, int C, int N, int S, int U, int J,
                  int T, float rho, Modem md, float2* x_hat, uint8_t* hard) {
    if (!cg_tc_ok(UP, J, N, C, S)) return false;
    CgTcArgs a{};
    a.N = N; a.C = C; a.S = S; a.U = U; a.T = T; a.rho = rho; a.md = md; a.x_hat = x_hat; a.hard = hard;
    a.S16 = S <= 16 ? 16 : (S + 31) / 32 * 32;              // antenna rows per cluster: whole 32-row groups
#ifndef DBP_CGT_RMIN
#define DBP_CGT_RMIN 32
#endif
    a.R = std::max(DBP_CGT_RMIN, a.S16);                    // rows per stage: 32 (1 or 2 clusters) or 64
    a.CB = a.R / a.S16;                                     // clusters per stage
    a.nstages = (C + a.CB - 1) / a.CB;                      // clusters >= C zero-filled by the TMA
    CUtensorMap tmH{}, tmY{};
    if (!make_map4(&tmH, H, U, S, N, C, 16, a.S16, 1, a.CB, true)) return false;
    if (!make_map4(&tmY, y, S, J, N, C, a.S16, J, 1, a.CB)) return false;
    if (J > 1) {
        CgTcjArgs aj{a, J};
        const size_t smem = 1024 + CGT_WARPS * cgtcj_warp_bytes(a.R, J);
        const int ks = a.nstages >= 8 ? 2 : 1;
        auto k = ks == 2 ? k_cg_tcj<2> : k_cg_tcj<1>;
        if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
            cudaGetLastError();
            return false;
        }
        if (!launch_pdl(k, (N + CGT_WARPS / ks - 1) / (CGT_WARPS / ks), CGT_WARPS * 32, smem, L, tmH, tmY, aj))
            return false;
        L.count(1);
        return true;
    }
    const size_t smem = cgtc_smem(a.R);
    const int ks = a.nstages >= 8 ? 2 : 1;                 // K split only when each warp keeps >= 4 stages
    auto k = ks == 2 ? k_cg_tc<2> : k_cg_tc<1>;
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    if (!launch_pdl(k, (N + CGT_WARPS / ks - 1) / (CGT_WARPS / ks), CGT_WARPS * 32, smem, L, tmH, tmY, a)) return false;
    L.count(1);
    return true;
}

}  // namespace dbp
