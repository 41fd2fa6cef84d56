// dbp_ss.cu -- the S x S forms of Alg. 1 and Alg. 3: for clusters with
// fewer antennas than users (S < U) the paper inverts an S x S matrix per cluster instead of
// the U x U one (Woodbury, P275-280, P482-488):
//
//   ADMM-UL (Alg. 1 lines 3-5, 13):  A_c = H_c H_c^H + rho I_S,  y^reg_c = H_c^H A_c^{-1} y_c,
//            z_c = y^reg_c + v - H_c^H A_c^{-1} H_c v,  v = s - lambda_c          (eq. (4), P278)
//   ADMM-DL (Alg. 3 lines 3-4, 9, 17): A_c = H_c^H H_c + rho^{-1} I_S,
//            x_c = A_c^{-1} H_c^H (z_c + lambda_c)                                   (P480-481)
//
// (H_c is the uplink [S][U] block in Alg. 1 and the downlink H^d_c [U][S] in Alg. 3.)  The
// iteration then applies three matrix-vector products per cluster (H_c, A_c^{-1}, H_c^H;
// Table I P584-586) instead of one.  Results equal the U x U forms up to rounding (reading 7).
//
// Layout: one warp per (cluster, subcarrier) pair, lane i holds index i of every vector
// (S- and U-indexed, both <= 32) and row i of A_c^{-1} (SP = S padded to 4/8/16/32; padded
// rows are identity rows, exactly decoupled).  H_c is staged in the warp's shared memory.
// Iterations: one launch per consensus round (CTA = one subcarrier, its warps walk the rank's
// clusters; the warps' partial sums are added in fixed order -- deterministic), the NCCL
// allreduce of the partial sums in between at world > 1, exactly as the U x U split path.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "dbp_device.cuh"
#include "dbp_internal.h"
#include "dbp_lanerow.cuh"

namespace dbp {

constexpr int SS_WARPS = 4;

// H_c of pair p into the warp's staging buffer hs: UL [S][U] (row s = antenna), DL [U][S].
__device__ __forceinline__ void ss_stage_h(float2* hs, const float2* __restrict__ H, size_t p, int S, int U, int lane) {
    const float2* src = H + p * (size_t)S * U;
    for (int e = lane; e < S * U; e += 32) hs[e] = __ldg(src + e);
    DBP_SYNCWARP();
}

// u = M v for the UL block (S x U, row-major in hs): lane i < S returns (H v)_i.
__device__ __forceinline__ float2 ss_h_mul(const float2* hs, const float2* vs, int S, int U, int i, bool dl) {
    float2 acc = make_float2(0.f, 0.f);
    if (i < (dl ? U : S))
        for (int k = 0; k < (dl ? S : U); ++k) c_fma(acc, hs[i * (dl ? S : U) + k], vs[k]);
    return acc;
}
// lane j < U (UL) / S (DL): (H^H t)_j
__device__ __forceinline__ float2 ss_hh_mul(const float2* hs, const float2* ts, int S, int U, int j, bool dl) {
    float2 acc = make_float2(0.f, 0.f);
    if (j < (dl ? S : U))
        for (int k = 0; k < (dl ? U : S); ++k) c_fmac(acc, hs[k * (dl ? S : U) + j], ts[k]);
    return acc;
}
// lane i < SP: (A^{-1} m)_i with row i of A^{-1} in R and m published in ms
template <int SP>
__device__ __forceinline__ float2 ss_ainv_mul(const float2 (&R)[SP], const float2* ms, int i) {
    float2 acc = make_float2(0.f, 0.f);
    if (i < SP) {
#pragma unroll
        for (int k = 0; k < SP; ++k) c_fma(acc, R[k], ms[k]);
    }
    return acc;
}

template <int SP>
__device__ __forceinline__ void ss_load_ainv(float2 (&R)[SP], const float2* __restrict__ Ap, int i) {
    if (i < SP) {
        load_herm_row<SP>(Ap, i, R);
    } else {
#pragma unroll
        for (int k = 0; k < SP; ++k) R[k] = make_float2(0.f, 0.f);
    }
}


// ---------------------------------------------------------------- preprocessing
// A^{-1} (packed lower) and, UL, y^reg_j = H^H A^{-1} y_j.
template <int SP, bool DL>
__global__ void __launch_bounds__(SS_WARPS * 32) k_ss_pre(SsArgs a) {
    extern __shared__ __align__(16) float2 ssm[];
    DBP_POISON_SMEM(ssm);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float2* hs = ssm + warp * (32 * 32 + 64);
    float2* vl = hs + 32 * 32;                       // [32] vector line
    float2* pr = vl + 32;                            // [32] pivot row (gj_invert)
    const long npairs = (long)a.C_loc * a.N;
    const int S = a.S, U = a.U;
    for (long p = (long)blockIdx.x * SS_WARPS + warp; p < npairs; p += (long)gridDim.x * SS_WARPS) {
        ss_stage_h(hs, a.H, (size_t)p, S, U, lane);
        // row i of A: UL sum_u H[i][u] conj(H[k][u]); DL sum_u conj(H[u][i]) H[u][k]; + delta I; padded rows = e_i
        float2 R[SP];
        const int i = lane;
#pragma unroll
        for (int k = 0; k < SP; ++k) {
            float2 acc = make_float2(0.f, 0.f);
            if (i < S && k < S) {
                if (DL) {
                    for (int u = 0; u < U; ++u) c_fmac(acc, hs[u * S + i], hs[u * S + k]);
                } else {
                    for (int u = 0; u < U; ++u) c_fmacb(acc, hs[i * U + u], hs[k * U + u]);
                }
            }
            if (k == i) acc = make_float2((i < S ? acc.x + a.delta : 1.f), 0.f);
            R[k] = acc;
        }
        const bool ok = gj_invert<SP>(R, pr, i);     // lanes >= SP hold zero rows and never publish
        if (!ok) atomicOr(a.flag, 1);
        float2* Ap = a.Ainv + (size_t)p * tri(SP);
        if (i < SP)
            for (int k = 0; k <= i; ++k) Ap[pidx(i, k)] = R[k];
        if (!DL) {
            for (int j = 0; j < a.J; ++j) {
                vl[lane] = i < S ? a.y[((size_t)p * a.J + j) * S + i] : make_float2(0.f, 0.f);
                DBP_SYNCWARP();
                const float2 t = ss_ainv_mul<SP>(R, vl, i);      // A^{-1} y_j
                DBP_SYNCWARP();
                vl[lane] = t;
                DBP_SYNCWARP();
                const float2 yr = ss_hh_mul(hs, vl, S, U, lane, false);                 // H^H (A^{-1} y_j)
                if (lane < a.UPW) a.yreg[((size_t)p * a.J + j) * a.UPW + lane] = yr;
                DBP_SYNCWARP();
            }
        }
        DBP_SYNCWARP();
    }
}

// ---------------------------------------------------------------- ADMM-UL round
// step 1: z = y^reg, lambda = 0, w = z (Alg. 1 line 10); step t >= 2: s = prox(w^(t-1)) from the
// allreduced partial sums, lines 12-17 with line 13's S x S form; the new partial sum
// sum_{c local} w_c replaces wbuf (the CTA owns subcarrier n).
template <int SP>
__global__ void __launch_bounds__(SS_WARPS * 32) k_ss_ul_it(SsArgs a) {
    extern __shared__ __align__(16) float2 ssm[];
    DBP_POISON_SMEM(ssm);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n = blockIdx.x, J = a.J, S = a.S, U = a.U;
    float2* Sv = ssm;                                 // [J][32] s^(t-1)
    float2* Wp = Sv + J * 32;                         // [WARPS][J][32] per-warp partials
    float2* hs = Wp + SS_WARPS * J * 32 + warp * (32 * 32 + 64);
    float2* vl = hs + 32 * 32;
    float2* tl = vl + 32;
    for (int e = threadIdx.x; e < J * 32; e += blockDim.x) {
        const int j = e / 32, u = e % 32;
        Sv[e] = (a.step > 1 && u < U) ? prox(a.wbuf[((size_t)n * J + j) * a.UPW + u], a.px) : make_float2(0.f, 0.f);
    }
    for (int e = lane; e < J * 32; e += 32) Wp[warp * J * 32 + e] = make_float2(0.f, 0.f);
    DBP_SYNCTHREADS();
    for (int c = warp; c < a.C_loc; c += SS_WARPS) {
        const size_t p = (size_t)c * a.N + n;
        float2 R[SP];
        if (a.step > 1) {
            ss_stage_h(hs, a.H, p, S, U, lane);
            ss_load_ainv<SP>(R, a.Ainv + p * tri(SP), lane);
        }
        for (int j = 0; j < J; ++j) {
            const bool own = lane < a.UPW;
            const size_t o = (p * J + j) * a.UPW + (own ? lane : 0);
            const float2 yr = own ? a.yreg[o] : make_float2(0.f, 0.f);
            float2 z, lam;
            if (a.step == 1) {
                z = yr;
                lam = make_float2(0.f, 0.f);
            } else {
                const float2 s = Sv[j * 32 + lane];
                lam = own ? c_add(a.lam[o], c_scale(c_sub(a.st[o], s), a.gamma)) : make_float2(0.f, 0.f);   // line 12
                const float2 v = lane < U ? c_sub(s, lam) : make_float2(0.f, 0.f);
                vl[lane] = v;
                DBP_SYNCWARP();
                const float2 m = ss_h_mul(hs, vl, S, U, lane, false);                  // H v
                DBP_SYNCWARP();
                tl[lane] = m;
                DBP_SYNCWARP();
                const float2 t = ss_ainv_mul<SP>(R, tl, lane);                        // A^{-1} H v
                DBP_SYNCWARP();
                vl[lane] = t;
                DBP_SYNCWARP();
                const float2 q = ss_hh_mul(hs, vl, S, U, lane, false);                 // H^H A^{-1} H v
                DBP_SYNCWARP();
                z = lane < U ? c_sub(c_add(yr, v), q) : make_float2(0.f, 0.f);         // line 15 (S <= U form)
            }
            if (own) {
                a.lam[o] = lam;
                a.st[o] = z;
            }
            Wp[(warp * J + j) * 32 + lane] = c_add(Wp[(warp * J + j) * 32 + lane], c_add(z, lam));   // line 17
        }
    }
    DBP_SYNCTHREADS();
    for (int e = threadIdx.x; e < J * a.UPW; e += blockDim.x) {                        // fixed warp order
        const int j = e / a.UPW, u = e % a.UPW;
        float2 acc = make_float2(0.f, 0.f);
        for (int w = 0; w < SS_WARPS; ++w) acc = c_add(acc, Wp[(w * J + j) * 32 + u]);
        a.wbuf[(size_t)n * J * a.UPW + e] = acc;
    }
}

// ---------------------------------------------------------------- ADMM-DL round
// step 0: z^(1) = a0 s, lambda = 0, x^(1) = A^{-1} H^H z (lines 8-9); if T > 1 also
// m^(1) = H x, w^(1) = m - lambda (lines 11-12) into wbuf, else x^(1) is the output.
// step t = 2..T: W = wbuf (allreduced), lines 14-15 (Lemma 2 for eps > 0), x^(t) (line 17);
// t < T: m^(t), w^(t) into wbuf; t = T: x^(T) is the output (P525).
template <int SP>
__global__ void __launch_bounds__(SS_WARPS * 32) k_ss_dl_it(SsArgs a) {
    extern __shared__ __align__(16) float2 ssm[];
    DBP_POISON_SMEM(ssm);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n = blockIdx.x, J = a.J, S = a.S, U = a.U;
    const bool last = a.step == a.T || (a.step == 0 && a.T == 1);
    float2* Sd = ssm;                                 // [J][32] s - W (or s at step 0)
    float* fj = reinterpret_cast<float*>(Sd + J * 32);   // [J] Lemma-2 factor (padded to 32 floats)
    float2* Wv = Sd + J * 32 + 16;                    // [J][32] W
    float2* Wp = Wv + J * 32;                         // [WARPS][J][32]
    float2* hs = Wp + SS_WARPS * J * 32 + warp * (32 * 32 + 64);
    float2* vl = hs + 32 * 32;
    float2* tl = vl + 32;
    for (int e = threadIdx.x; e < J * 32; e += blockDim.x) {
        const int j = e / 32, u = e % 32;
        const float2 sv = u < U ? a.s[((size_t)n * J + j) * U + u] : make_float2(0.f, 0.f);
        const float2 W = (a.step > 0 && u < U) ? a.wbuf[((size_t)n * J + j) * a.UPW + u] : make_float2(0.f, 0.f);
        Wv[e] = W;
        Sd[e] = a.step > 0 ? c_sub(sv, W) : sv;
    }
    DBP_SYNCTHREADS();
    if (a.step > 0) {
        for (int j = warp; j < J; j += SS_WARPS) {     // ||s - W|| per symbol (Lemma 2, P538)
            float nrm2 = c_norm2(Sd[j * 32 + lane]);
            for (int o = 16; o; o >>= 1) nrm2 += __shfl_xor_sync(0xffffffffu, nrm2, o);
            if (lane == 0) fj[j] = lemma2_scale(nrm2, a.eps, a.inv_c);
        }
    }
    for (int e = lane; e < J * 32; e += 32) Wp[warp * J * 32 + e] = make_float2(0.f, 0.f);
    DBP_SYNCTHREADS();
    for (int c = warp; c < a.C_loc; c += SS_WARPS) {
        const size_t p = (size_t)c * a.N + n;
        float2 R[SP];
        ss_stage_h(hs, a.H, p, S, U, lane);
        ss_load_ainv<SP>(R, a.Ainv + p * tri(SP), lane);
        for (int j = 0; j < J; ++j) {
            const bool own = lane < a.UPW;
            const size_t o = (p * J + j) * a.UPW + (own ? lane : 0);
            float2 q, lam;
            if (a.step == 0) {
                q = c_scale(Sd[j * 32 + lane], a.a0);                                  // z^(1) + lambda^(1)
                lam = make_float2(0.f, 0.f);
            } else {
                const float2 m = own ? a.st[o] : make_float2(0.f, 0.f);
                const float2 l0 = own ? a.lam[o] : make_float2(0.f, 0.f);
                const float2 w = c_sub(m, l0);                                          // line 12 (local)
                const float2 z = c_add(w, c_scale(Sd[j * 32 + lane], fj[j]));          // line 14
                lam = c_sub(l0, c_scale(c_sub(m, z), a.gamma));                        // line 15
                q = lane < U ? c_add(z, lam) : make_float2(0.f, 0.f);
            }
            vl[lane] = q;
            DBP_SYNCWARP();
            const float2 hq = ss_hh_mul(hs, vl, S, U, lane, true);                      // H^H q (S)
            DBP_SYNCWARP();
            tl[lane] = hq;
            DBP_SYNCWARP();
            const float2 x = ss_ainv_mul<SP>(R, tl, lane);                              // line 17 (S <= U form)
            DBP_SYNCWARP();
            if (last) {
                if (lane < S) a.x[((size_t)p * J + j) * S + lane] = x;
            } else {
                vl[lane] = lane < S ? x : make_float2(0.f, 0.f);
                DBP_SYNCWARP();
                const float2 m = ss_h_mul(hs, vl, S, U, lane, true);                    // line 11: m = H x
                DBP_SYNCWARP();
                if (own) {
                    a.st[o] = m;
                    a.lam[o] = lam;
                }
                Wp[(warp * J + j) * 32 + lane] = c_add(Wp[(warp * J + j) * 32 + lane], c_sub(m, lam));  // line 12
            }
        }
    }
    if (last) return;
    DBP_SYNCTHREADS();
    for (int e = threadIdx.x; e < J * a.UPW; e += blockDim.x) {
        const int j = e / a.UPW, u = e % a.UPW;
        float2 acc = make_float2(0.f, 0.f);
        for (int w = 0; w < SS_WARPS; ++w) acc = c_add(acc, Wp[(w * J + j) * 32 + u]);
        a.wbuf[(size_t)n * J * a.UPW + e] = acc;
    }
}

static int ss_pad(int S) { return S <= 4 ? 4 : S <= 8 ? 8 : S <= 16 ? 16 : 32; }
size_t ss_iter_smem(int J) { return ((size_t)J * 32 * (2 + SS_WARPS) + 16 + (size_t)SS_WARPS * (32 * 32 + 64)) * 8; }
static size_t ss_pre_smem() { return (size_t)SS_WARPS * (32 * 32 + 64) * 8; }

template <typename K>
static cudaError_t ss_smem_attr(K k, size_t smem) {
    if (smem > 48 * 1024) return cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    return cudaSuccess;
}

cudaError_t launch_ss_pre(const LaunchCtx& L, bool dl, SsArgs a) {
    const long npairs = (long)a.C_loc * a.N;
    if (npairs <= 0) return cudaSuccess;
    const int grid = (int)std::min<long>((npairs + SS_WARPS - 1) / SS_WARPS, 148L * 16);
    const size_t smem = ss_pre_smem();
    cudaError_t e = cudaSuccess;
    DBP_DISPATCH_UP(ss_pad(a.S),
        auto k = dl ? k_ss_pre<UPc, true> : k_ss_pre<UPc, false>;
        e = ss_smem_attr(k, smem);
        if (e == cudaSuccess) k<<<grid, SS_WARPS * 32, smem, L.stream>>>(a));
    L.count(1);
    return e != cudaSuccess ? e : cudaGetLastError();
}

cudaError_t launch_ss_it(const LaunchCtx& L, bool dl, SsArgs a) {
    if (a.N <= 0) return cudaSuccess;
    const size_t smem = ss_iter_smem(a.J);
    cudaError_t e = cudaSuccess;
    DBP_DISPATCH_UP(ss_pad(a.S),
        auto k = dl ? k_ss_dl_it<UPc> : k_ss_ul_it<UPc>;
        e = ss_smem_attr(k, smem);
        if (e == cudaSuccess) k<<<a.N, SS_WARPS * 32, smem, L.stream>>>(a));
    L.count(1);
    return e != cudaSuccess ? e : cudaGetLastError();
}

}  // namespace dbp
