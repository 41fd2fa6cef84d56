// dbp_tc.cuh -- the per-pair Gram (+ matched filter) on the tensor cores, for UP = 16
// (G_c = H_c^H H_c (P295, P391), B_c = H_c H_c^H (P503),
// H_c^H y_c (P296)).  In k_fused this stays behind the build knob DBP_FZ_TC (off: measured slower
// than the folded FP32 Gram at K = S = 32); the FP16 helpers below (mma_f16, f16x2,
// tc16_load, TC_NEG2) also carry the long-K cluster-summed Grams of CG, which are the default
// (dbp_cgtc.cu, dbp_cgg.cu).
//
// One warp computes one pair with mma.sync m16n8k8 TF32 (the warp-level tensor path; 242
// TFLOP/s measured on B200, scripts/micro/tc_gram.cu) in "3xTF32": every fp32 operand v is
// split exactly into hi = v with the low 13 mantissa bits cleared (a TF32 value) and
// lo = v - hi (exact in fp32; the tensor core keeps its top 19 bits), and
// hi*hi + hi*lo + lo*hi is accumulated in fp32 -- the dropped lo*lo term and lo's
// truncation are ~2^-22 relative, so the Gram matches an fp32 FMA Gram (measured 6e-7
// relative to fp64, vs 1.5e-4 for plain TF32).  Scale-free (TF32 keeps the fp32 exponent).
//
// Real form: with A[u][k] = (Re or Im) of h_{k,u} over the K index k = antenna (a K8 step
// is 8 antennas, taken once for the real and once for the imaginary parts),
//   Re G = A_re^T A_re + A_im^T A_im,   Im G = A_re^T A_im - A_im^T A_re  (UL: G = H^H H),
// so M = 16 users, N = 32 ([Re G | Im G], four n8 tiles), and the B operand of the Re tiles
// is A^T itself: every fragment is built from the same 4 complex values per lane and K8 step,
//   v[e1][e2] = h(user g + 8 e1, antenna 8 kk + 2 t + e2),   g = lane / 4, t = lane % 4
// (K index t <-> antenna 2t, t + 4 <-> 2t + 1: the 8 lanes of a quarter-warp then read 8
// distinct 16-B chunks of the 128B-swizzled TMA stage, see below).  A fifth n8 tile carries
// the matched filter: columns [y_re; y_im] and [y_im; -y_re] give Re and Im of H^H y.
//
// Stage layouts in shared memory (TMA, CU_TENSOR_MAP_SWIZZLE_128B, 1024-B aligned):
//   UL: H_c [S8 antennas][16 users] (128-B rows: chunk c of row s at c ^ (s & 7)), then
//       y_c [S8] unswizzled;
//   DL: H^d_c as ceil(S/16) boxes of [16 users][16 antennas] (2 KB each; chunk c of row u
//       at c ^ (u & 7)).  B = H H^H has Im of the opposite sign (conjugate of the UL form).
#pragma once

#include "dbp_device.cuh"

namespace dbp {

__device__ __forceinline__ void mma_tf32(float (&d)[4], unsigned a0, unsigned a1, unsigned a2, unsigned a3,
                                         unsigned b0, unsigned b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// Exact split v = hi + lo, hi a TF32 value (low 13 mantissa bits cleared).
__device__ __forceinline__ void tc_split(float v, unsigned& hi, unsigned& lo) {
    hi = __float_as_uint(v) & 0xffffe000u;
    lo = __float_as_uint(v - __uint_as_float(hi));
}

constexpr unsigned TC_NEG = 0x80000000u;

// Gram (+ matched filter) of one pair from its TMA stage; acc[0..1] Re tiles (columns
// 0-7, 8-15), acc[2..3] Im tiles, acc[4] matched filter (columns 0 = Re, 1 = Im).
// nkk = number of K8 steps (ceil(S / 8)); antennas >= S are zero-filled by the TMA.
// (kk0, kk1: the K8 steps to take, accumulate: add to acc instead of starting from zero, yoff: byte
// offset of y in the stage -- a longer K, e.g. several clusters' antennas stacked as rows, is the
// same loop; see dbp_cgtc.cu)
template <bool DL, bool MF>
__device__ __forceinline__ void tc_gram(float (&acc)[5][4], const unsigned char* stage, int nkk, int g, int t,
                                        int kk0 = 0, int kk1 = -1, bool accumulate = false, int yoff = -1) {
    if (!accumulate) {
#pragma unroll
        for (int i = 0; i < 5; ++i)
#pragma unroll
            for (int e = 0; e < 4; ++e) acc[i][e] = 0.f;
    }
    if (kk1 < 0) kk1 = nkk;
    const float2* yv = reinterpret_cast<const float2*>(stage + (yoff >= 0 ? yoff : nkk * 8 * 128));   // UL: y after H
#pragma unroll 2
    for (int kk = kk0; kk < kk1; ++kk) {
        float2 v[2][2];
        if (DL) {
            // box kk/2, row u, the 16-B chunk holding antennas 8(kk&1) + 2t, +1
#pragma unroll
            for (int e1 = 0; e1 < 2; ++e1) {
                const int u = g + 8 * e1;
                const float4 q = *reinterpret_cast<const float4*>(stage + (kk >> 1) * 2048 + u * 128 +
                                                                  (((4 * (kk & 1) + t) ^ g) << 4));
                v[e1][0] = make_float2(q.x, q.y);
                v[e1][1] = make_float2(q.z, q.w);
            }
        } else {
#pragma unroll
            for (int e2 = 0; e2 < 2; ++e2) {
                const int s = 8 * kk + 2 * t + e2;
#pragma unroll
                for (int e1 = 0; e1 < 2; ++e1) {
                    const int u = g + 8 * e1;
                    v[e1][e2] = *reinterpret_cast<const float2*>(stage + s * 128 + (((u >> 1) ^ (s & 7)) << 4) +
                                                                 ((u & 1) << 3));
                }
            }
        }
        // fragment order a0 (user g, k t), a1 (g + 8, t), a2 (g, t + 4), a3 (g + 8, t + 4)
        unsigned rh[4], rl[4], ih[4], il[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const float2 x = v[e & 1][e >> 1];
            tc_split(x.x, rh[e], rl[e]);
            tc_split(x.y, ih[e], il[e]);
        }
        unsigned yrh[2], yrl[2], yih[2], yil[2];
        if (MF) {
            // B[k][col g] of the matched-filter tile: col 0 = (y_re | y_im), col 1 = (y_im | -y_re)
            // over the (re | im) K steps; b0 <- antenna 2t, b1 <- 2t + 1; columns >= 2 are zero
            const float4 yy = *reinterpret_cast<const float4*>(yv + 8 * kk + 2 * t);
            const float re0 = g == 0 ? yy.x : (g == 1 ? yy.y : 0.f), re1 = g == 0 ? yy.z : (g == 1 ? yy.w : 0.f);
            const float im0 = g == 0 ? yy.y : (g == 1 ? -yy.x : 0.f), im1 = g == 0 ? yy.w : (g == 1 ? -yy.z : 0.f);
            tc_split(re0, yrh[0], yrl[0]);
            tc_split(re1, yrh[1], yrl[1]);
            tc_split(im0, yih[0], yil[0]);
            tc_split(im1, yih[1], yil[1]);
        }
        // three passes: (A hi, B hi), (A hi, B lo), (A lo, B hi)
#pragma unroll
        for (int pass = 0; pass < 3; ++pass) {
            const unsigned* Ar = pass == 2 ? rl : rh;
            const unsigned* Ai = pass == 2 ? il : ih;
            const unsigned* Br = pass == 1 ? rl : rh;
            const unsigned* Bi = pass == 1 ? il : ih;
            mma_tf32(acc[0], Ar[0], Ar[1], Ar[2], Ar[3], Br[0], Br[2]);
            mma_tf32(acc[0], Ai[0], Ai[1], Ai[2], Ai[3], Bi[0], Bi[2]);
            mma_tf32(acc[1], Ar[0], Ar[1], Ar[2], Ar[3], Br[1], Br[3]);
            mma_tf32(acc[1], Ai[0], Ai[1], Ai[2], Ai[3], Bi[1], Bi[3]);
            mma_tf32(acc[2], Ar[0], Ar[1], Ar[2], Ar[3], Bi[0], Bi[2]);
            mma_tf32(acc[2], Ai[0], Ai[1], Ai[2], Ai[3], Br[0] ^ TC_NEG, Br[2] ^ TC_NEG);
            mma_tf32(acc[3], Ar[0], Ar[1], Ar[2], Ar[3], Bi[1], Bi[3]);
            mma_tf32(acc[3], Ai[0], Ai[1], Ai[2], Ai[3], Br[1] ^ TC_NEG, Br[3] ^ TC_NEG);
            if (MF) {
                const unsigned* Yr = pass == 1 ? yrl : yrh;
                const unsigned* Yi = pass == 1 ? yil : yih;
                mma_tf32(acc[4], Ar[0], Ar[1], Ar[2], Ar[3], Yr[0], Yr[1]);
                mma_tf32(acc[4], Ai[0], Ai[1], Ai[2], Ai[3], Yi[0], Yi[1]);
            }
        }
    }
}

// Lower triangle of the pair's Gram (DL: conjugated to B = H H^H) into a packed [TRI] line,
// and (MF) H^H y into a [16] line.  D fragment: c0 (row g, col 2t), c1 (g, 2t+1), c2 (g+8, 2t),
// c3 (g+8, 2t+1) of each n8 tile; columns 8h + 2t + cc of tile h (Re) and 2 + h (Im).
template <bool DL, bool MF>
__device__ __forceinline__ void tc_store(const float (&acc)[5][4], float2* gtri, float2* mfl, int g, int t) {
    const float sg = DL ? -1.f : 1.f;
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int e1 = 0; e1 < 2; ++e1)
#pragma unroll
            for (int cc = 0; cc < 2; ++cc) {
                const int r = g + 8 * e1, col = 8 * h + 2 * t + cc;
                if (col <= r) gtri[pidx(r, col)] = make_float2(acc[h][2 * e1 + cc], sg * acc[2 + h][2 * e1 + cc]);
            }
    if (MF && t == 0) {
        mfl[g] = make_float2(acc[4][0], acc[4][1]);
        mfl[g + 8] = make_float2(acc[4][2], acc[4][3]);
    }
}


// ---------------------------------------------------------------------------------------------
// FP16 variant (DBP_FZ_TC == 2): mma.sync m16n8k16 f16 -> f32 (485 TFLOP/s measured, twice TF32)
// with two passes instead of three.  The pair is first scaled by an exact power of two so its
// largest |Re|, |Im| lies in [1, 2) (warp max; fp16 then keeps the split normal down to 2^-14 of
// it -- scale-free like TF32).  v = hi + lo with hi = v with the low 13 mantissa bits cleared
// (exactly an fp16 value) and lo = v - hi.  Since G = hi^H hi + hi^H lo + lo^H hi (dropping
// lo^H lo, ~2^-22) is Z + Z^H with Z = 0.5 hi^H hi + hi^H lo, the tensor cores form Z (A = hi,
// B = 0.5 hi then B = lo: two passes) and G_rc = Z_rc + conj(Z_cr) is formed through a per-warp
// [16][17] scratch.  The matched filter H^H y (16 values) runs on the FP32 cores from the same
// fragments (unscaled), summed over the 4 lanes of a quad.
//
// K16 step kk covers antennas 16 kk .. 16 kk + 15 (K index = antenna); lane (g, t) holds
//   v[uh][kh][e] = h(user g + 8 uh, antenna 16 kk + 8 kh + 2 t + e),
// the A fragments a0 = {v[0][0][0..1]}, a1 = {v[1][0][..]}, a2 = {v[0][1][..]}, a3 = {v[1][1][..]}
// (Re and Im parts separately), and -- B of the Re tiles being A^T -- all B fragments.
__device__ __forceinline__ void mma_f16(float (&d)[4], unsigned a0, unsigned a1, unsigned a2, unsigned a3,
                                        unsigned b0, unsigned b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ unsigned f16x2(float lo_half, float hi_half) {
    unsigned r;
    asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi_half), "f"(lo_half));
    return r;
}
constexpr unsigned TC_NEG2 = 0x80008000u;

// Stage reads of one K16 step (see the layouts above).
template <bool DL>
__device__ __forceinline__ void tc16_load(float2 (&v)[2][2][2], const unsigned char* stage, int kk, int g, int t) {
    if (DL) {
#pragma unroll
        for (int uh = 0; uh < 2; ++uh)
#pragma unroll
            for (int kh = 0; kh < 2; ++kh) {
                const float4 q = *reinterpret_cast<const float4*>(stage + kk * 2048 + (g + 8 * uh) * 128 +
                                                                  (((4 * kh + t) ^ g) << 4));
                v[uh][kh][0] = make_float2(q.x, q.y);
                v[uh][kh][1] = make_float2(q.z, q.w);
            }
    } else {
#pragma unroll
        for (int kh = 0; kh < 2; ++kh)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int s = 16 * kk + 8 * kh + 2 * t + e;
#pragma unroll
                for (int uh = 0; uh < 2; ++uh) {
                    const int u = g + 8 * uh;
                    v[uh][kh][e] = *reinterpret_cast<const float2*>(stage + s * 128 + (((u >> 1) ^ (s & 7)) << 4) +
                                                                    ((u & 1) << 3));
                }
            }
    }
}

// G (lower triangle, packed) and, UL, H^H y of one pair.  zs: per-warp [16][17] float2 scratch.
// nk16 = ceil(S / 16) K16 steps (antennas >= S zero-filled by the TMA).
template <bool DL, bool MF>
__device__ __forceinline__ void tc16_gram_pair(const unsigned char* stage, int nk16, float2* gtri, float2* mfl,
                                               float2* zs, int g, int t, int lane) {
    // pass 0: the pair's scale (exact power of two)
    float mx = 0.f;
    for (int kk = 0; kk < nk16; ++kk) {
        float2 v[2][2][2];
        tc16_load<DL>(v, stage, kk, g, t);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const float2 x = v[i >> 2][(i >> 1) & 1][i & 1];
            mx = fmaxf(mx, fmaxf(fabsf(x.x), fabsf(x.y)));
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    const int ex = mx > 0.f ? ((__float_as_int(mx) >> 23) & 0xff) - 127 : 0;
    const float sc = __int_as_float((127 - ex) << 23);                 // 2^-ex: max -> [1, 2)
    float acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int e = 0; e < 4; ++e) acc[i][e] = 0.f;
    f2x mf[2] = {0ull, 0ull};
    const float2* yv = reinterpret_cast<const float2*>(stage + nk16 * 16 * 128);   // UL: y after H
    for (int kk = 0; kk < nk16; ++kk) {
        float2 v[2][2][2];
        tc16_load<DL>(v, stage, kk, g, t);
        if (MF) {
            // conj(h_su) y_s over this lane's 8 (antenna, user) values, FP32, unscaled
#pragma unroll
            for (int kh = 0; kh < 2; ++kh) {
                const float4 yy = *reinterpret_cast<const float4*>(yv + 16 * kk + 8 * kh + 2 * t);
#pragma unroll
                for (int uh = 0; uh < 2; ++uh) {
                    x2_cmac(mf[uh], v[uh][kh][0], yy.x, yy.y);
                    x2_cmac(mf[uh], v[uh][kh][1], yy.z, yy.w);
                }
            }
        }
        // fragments: index f = uh + 2 kh  (a0: uh 0 kh 0, a1: uh 1 kh 0, a2: uh 0 kh 1, a3: uh 1 kh 1)
        unsigned rh[4], ih[4], rq[4], iq[4], rl[4], il[4];
#pragma unroll
        for (int f = 0; f < 4; ++f) {
            const int uh = f & 1, kh = f >> 1;
            float hr[2], hi_[2], lr[2], li[2];
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const float xr = v[uh][kh][e].x * sc, xi = v[uh][kh][e].y * sc;
                hr[e] = __uint_as_float(__float_as_uint(xr) & 0xffffe000u);
                hi_[e] = __uint_as_float(__float_as_uint(xi) & 0xffffe000u);
                lr[e] = xr - hr[e];
                li[e] = xi - hi_[e];
            }
            rh[f] = f16x2(hr[0], hr[1]);
            ih[f] = f16x2(hi_[0], hi_[1]);
            rq[f] = f16x2(0.5f * hr[0], 0.5f * hr[1]);
            iq[f] = f16x2(0.5f * hi_[0], 0.5f * hi_[1]);
            rl[f] = f16x2(lr[0], lr[1]);
            il[f] = f16x2(li[0], li[1]);
        }
        // Z += hi^H (0.5 hi) + hi^H lo: Re tiles A_re B_re + A_im B_im, Im tiles A_re B_im - A_im B_re
#pragma unroll
        for (int pass = 0; pass < 2; ++pass) {
            const unsigned* Br = pass ? rl : rq;
            const unsigned* Bi = pass ? il : iq;
            mma_f16(acc[0], rh[0], rh[1], rh[2], rh[3], Br[0], Br[2]);
            mma_f16(acc[0], ih[0], ih[1], ih[2], ih[3], Bi[0], Bi[2]);
            mma_f16(acc[1], rh[0], rh[1], rh[2], rh[3], Br[1], Br[3]);
            mma_f16(acc[1], ih[0], ih[1], ih[2], ih[3], Bi[1], Bi[3]);
            mma_f16(acc[2], rh[0], rh[1], rh[2], rh[3], Bi[0], Bi[2]);
            mma_f16(acc[2], ih[0], ih[1], ih[2], ih[3], Br[0] ^ TC_NEG2, Br[2] ^ TC_NEG2);
            mma_f16(acc[3], rh[0], rh[1], rh[2], rh[3], Bi[1], Bi[3]);
            mma_f16(acc[3], ih[0], ih[1], ih[2], ih[3], Br[1] ^ TC_NEG2, Br[3] ^ TC_NEG2);
        }
    }
    // G = Z + Z^H through the scratch (row stride 17: the transposed reads are 2-way at most)
    const float us = __int_as_float((127 + 2 * ex) << 23);                // 2^(2 ex)
    DBP_SYNCWARP();
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int e1 = 0; e1 < 2; ++e1)
#pragma unroll
            for (int cc = 0; cc < 2; ++cc)
                zs[(g + 8 * e1) * 17 + 8 * h + 2 * t + cc] = make_float2(acc[h][2 * e1 + cc], acc[2 + h][2 * e1 + cc]);
    DBP_SYNCWARP();
    const float sg = DL ? -1.f : 1.f;                                     // DL: B = H H^H = conj(UL form)
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int e1 = 0; e1 < 2; ++e1)
#pragma unroll
            for (int cc = 0; cc < 2; ++cc) {
                const int r = g + 8 * e1, c = 8 * h + 2 * t + cc;
                if (c <= r) {
                    const float2 zt = zs[c * 17 + r];
                    gtri[pidx(r, c)] = make_float2((acc[h][2 * e1 + cc] + zt.x) * us,
                                                   sg * (acc[2 + h][2 * e1 + cc] - zt.y) * us);
                }
            }
    if (MF) {
#pragma unroll
        for (int uh = 0; uh < 2; ++uh) {
            float2 m = upk2(mf[uh]);
#pragma unroll
            for (int o = 1; o < 4; o <<= 1) {
                m.x += __shfl_xor_sync(0xffffffffu, m.x, o);
                m.y += __shfl_xor_sync(0xffffffffu, m.y, o);
            }
            if (t == 0) mfl[g + 8 * uh] = m;
        }
    }
    (void)lane;
}

}  // namespace dbp
