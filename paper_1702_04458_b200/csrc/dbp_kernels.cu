// dbp_kernels.cu -- sm_100a kernels of libdbp and their launchers.
//
// Kernel map (SURVEY.md 8(a) rows -> kernels):
//   k_pre      a1-a3 / b1 / c1  per (cluster, subcarrier) pair: TMA bulk copy
//                               of H_c into shared memory, Hermitian Gram by
//                               warp-uniform 4x4 tile jobs, team Cholesky,
//                               triangular inverse X = L^{-1}, matched filter.
//   k_admm_it  a4-a7            ADMM-UL consensus iterations: split (one step
//                               per launch + NCCL between) or fused (all T
//                               iterations on chip, world == 1).
//   k_cg_gsum  b1 (sum)         per-GPU Gram sum G_loc = sum_c H_c^H H_c
//                               (Alg. 2 line 9 footnote, P416) + local y^MRC.
//   k_cg_it    b2-b5            replicated CG updates with shuffle allreduce
//                               dot products (P715), split or fused.
//   k_bf_it    c2-c4            ADMM-DL iterations in the exact m-form,
//                               split or fused, incl. the final x_c pass.
//   k_prox_out a7-a8            final prox + hard slicing of the split path.
//   k_slice                     stand-alone slicer (P210).
#include <cuda_runtime.h>
#include <stdint.h>

#include "dbp_device.cuh"
#include "dbp_internal.h"

namespace dbp {

// ============================================================ k_pre
// Per-pair preprocessing.  PRE_ADMM: B_c = H^H H + rho I -> X = L^{-1}, yreg
// = X^H X H^H y.  PRE_BF: B_c = H^d H^dH + rho^{-1} I -> X.  PRE_CG: per-pair
// Gram H^H H and matched filter H^H y (summed over clusters by k_cg_gsum).
enum { PRE_ADMM = PRE_ADMM_, PRE_BF = PRE_BF_, PRE_CG = PRE_CG_ };

template <int UP>
struct PreCfg {
    using Tl = Tiles<UP>;
    static constexpr int PPC = UP == 4 ? 128 : UP == 8 ? 64 : UP == 16 ? 16 : 8;  // pairs per CTA
    static constexpr int WOFF = PPC * Tl::NOFF / 32;
    static constexpr int WDIAG = PPC * Tl::NDIAG / 32;
    static constexpr int THREADS = 32 * (WOFF + WDIAG);
    static constexpr int TPP = THREADS / PPC;
    static_assert(PPC * Tl::NOFF % 32 == 0 && PPC * Tl::NDIAG % 32 == 0, "warp-uniform jobs");
    static_assert(32 % TPP == 0, "team inside a warp");
};

__host__ __device__ inline int tile_stride(int S, int U) { return ((S * U + 1) & ~1) + 2; }   // float2, 16 B aligned + pad
__host__ __device__ inline int ytile_stride(int S, int J) { return ((S * J + 1) & ~1) + 2; }

template <int UP>
size_t pre_smem_bytes(int S, int U, int J, int mode) {
    using PC = PreCfg<UP>;
    size_t b = 16;                                                   // mbarrier
    b += (size_t)PC::PPC * tile_stride(S, U) * 8;
    if (mode != PRE_BF) b += (size_t)PC::PPC * ytile_stride(S, J) * 8;
    b += (size_t)PC::PPC * tri(UP) * 8;                              // Lp
    b += (size_t)PC::PPC * 2 * UP * 8;                               // v, u
    return b;
}

template <int UP, bool DL, bool FULL, int MODE>
__global__ void __launch_bounds__(PreCfg<UP>::THREADS)
k_pre(const float2* __restrict__ H, const float2* __restrict__ y, int S, int U, int J, int npairs,
      float delta, float2* __restrict__ Xout, float2* __restrict__ vout, int* __restrict__ flag) {
    using PC = PreCfg<UP>;
    using Tl = Tiles<UP>;
    using RM = RowMap<UP, PC::TPP>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw);
    float2* tiles = reinterpret_cast<float2*>(smem_raw + 16);
    const int ts = tile_stride(S, U);
    float2* ytiles = tiles + (size_t)PC::PPC * ts;
    const int yts = (MODE != PRE_BF) ? ytile_stride(S, J) : 0;
    float2* Lp = ytiles + (size_t)PC::PPC * yts;
    float2* vec = Lp + (size_t)PC::PPC * tri(UP);

    const int tid = threadIdx.x;
    const long p0 = (long)blockIdx.x * PC::PPC;
    const int nvalid = (int)min((long)PC::PPC, (long)npairs - p0);
    const uint32_t hbytes = (uint32_t)(S * U * 8);
    const uint32_t ybytes = (uint32_t)(S * J * 8);
    const bool bulk = ((hbytes | ybytes) & 15u) == 0;

    // ---- stage H_c (and y_c) tiles: one TMA bulk copy per pair
    if (bulk) {
        if (tid == 0) { mbar_init(bar, 1); fence_mbar_init(); }
        __syncthreads();
        if (tid == 0) {
            uint32_t total = nvalid * hbytes + (MODE != PRE_BF ? nvalid * ybytes : 0u);
            mbar_arrive_expect_tx(bar, total);
            for (int i = 0; i < nvalid; ++i) {
                bulk_g2s(tiles + (size_t)i * ts, H + (size_t)(p0 + i) * S * U, hbytes, bar);
                if (MODE != PRE_BF) bulk_g2s(ytiles + (size_t)i * yts, y + (size_t)(p0 + i) * S * J, ybytes, bar);
            }
        }
        mbar_wait(bar, 0);
    } else {
        for (int i = 0; i < nvalid; ++i) {
            for (int e = tid; e < S * U; e += blockDim.x) tiles[(size_t)i * ts + e] = H[(size_t)(p0 + i) * S * U + e];
            if (MODE != PRE_BF)
                for (int e = tid; e < S * J; e += blockDim.x) ytiles[(size_t)i * yts + e] = y[(size_t)(p0 + i) * S * J + e];
        }
        __syncthreads();
    }

    // ---- Gram by tile jobs (warp-uniform job type)
    const int warp = tid >> 5, lane = tid & 31;
    if (warp < PC::WOFF) {
        const int job = warp * 32 + lane;
        const int pi = job / Tl::NOFF;
        int a, b;
        off_tile_coords(job % Tl::NOFF, a, b);
        float2 acc[16];
        gram_off<DL, FULL>(tiles + (size_t)pi * ts, S, U, a, b, acc);
        float2* L = Lp + (size_t)pi * tri(UP);
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                float2 g = acc[r * 4 + c];
                L[pidx(4 * a + r, 4 * b + c)] = DL ? c_conj(g) : g;
            }
    } else {
        const int job = (warp - PC::WOFF) * 32 + lane;
        const int pi = job / Tl::NDIAG;
        const int e = job % Tl::NDIAG;
        const int d0 = Tl::NB >= 2 ? 2 * e : 0;
        const int d1 = Tl::NB >= 2 ? 2 * e + 1 : -1;
        float2 acc[20];
        gram_diag<DL, FULL>(tiles + (size_t)pi * ts, S, U, d0, d1, acc);
        float2* L = Lp + (size_t)pi * tri(UP);
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            const int d = q ? d1 : d0;
            if (d < 0) continue;
#pragma unroll
            for (int r = 0; r < 4; ++r)
#pragma unroll
                for (int c = 0; c <= r; ++c) {
                    float2 g = acc[q * 10 + pidx(r, c)];
                    if (r == c) g = make_float2(g.x + delta, 0.f);
                    L[pidx(4 * d + r, 4 * d + c)] = DL ? c_conj(g) : g;
                }
        }
    }
    __syncthreads();

    // ---- per-pair team work
    const int pi = tid / PC::TPP;
    const int t = tid % PC::TPP;
    const bool valid = pi < nvalid;
    float2* L = Lp + (size_t)pi * tri(UP);
    float2* v = vec + (size_t)pi * 2 * UP;
    float2* u = v + UP;
    const long p = p0 + pi;

    if (MODE == PRE_CG) {
        // per-pair Gram out, matched filter out
        for (int e = t; e < tri(UP); e += PC::TPP)
            if (valid) Xout[(size_t)p * tri(UP) + e] = L[e];
    } else {
        bool ok = team_cholesky<UP, PC::TPP>(L, t);
        if (!ok && valid && t == 0) atomicOr(flag, 1);
        team_tri_inverse<UP, PC::TPP>(L, t);
        for (int e = t; e < tri(UP); e += PC::TPP)
            if (valid) Xout[(size_t)p * tri(UP) + e] = L[e];
    }
    if (MODE == PRE_BF) return;

    // matched filter mf = H^H y_j (owned rows), then yreg = X^H X mf (ADMM)
    const float2* Ht = tiles + (size_t)pi * ts;
    const float2* yt = ytiles + (size_t)pi * yts;
    for (int j = 0; j < J; ++j) {
        float2 mf[RM::NR];
#pragma unroll
        for (int k = 0; k < RM::NR; ++k) {
            const int r = RM::row(t, k);
            float2 acc = make_float2(0.f, 0.f);
            if (FULL || r < U)
                for (int s = RM::sub(t); s < S; s += RM::TR) c_fmac(acc, Ht[s * U + r], yt[j * S + s]);
            if (RM::TR > 1) {
#pragma unroll
                for (int o = 1; o < RM::TR; o <<= 1) {
                    acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
                    acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
                }
            }
            mf[k] = acc;
        }
        if (MODE == PRE_CG) {
            if (valid && RM::sub(t) == 0)
#pragma unroll
                for (int k = 0; k < RM::NR; ++k) vout[((size_t)p * J + j) * UP + RM::row(t, k)] = mf[k];
            continue;
        }
        __syncwarp();
        if (RM::sub(t) == 0)
#pragma unroll
            for (int k = 0; k < RM::NR; ++k) v[RM::row(t, k)] = mf[k];
        __syncwarp();
        float2 tmp[RM::NR];
        tri_mv<UP, PC::TPP>(L, v, t, tmp);
        __syncwarp();
        if (RM::sub(t) == 0)
#pragma unroll
            for (int k = 0; k < RM::NR; ++k) u[RM::row(t, k)] = tmp[k];
        __syncwarp();
        tri_mv_h<UP, PC::TPP>(L, u, t, tmp);
        if (valid && RM::sub(t) == 0)
#pragma unroll
            for (int k = 0; k < RM::NR; ++k) vout[((size_t)p * J + j) * UP + RM::row(t, k)] = tmp[k];
    }
}

// ============================================================ ADMM-UL iterations
// Thread layout: team of IT = UP/2 threads per pair, thread owns rows
// {g, UP-1-g}.  CTA = NT subcarriers x CCH clusters (one chunk), clusters
// looped in chunks when C_loc > CCH (split path).  Consensus partial sums
// over the CTA's clusters are taken in fixed cluster order (deterministic).
template <int UP>
struct ItCfg {
    static constexpr int IT = UP / 2;     // threads per pair
    using RM = RowMap<UP, IT>;
};



// One ADMM local update of Alg. 1 lines 12-18 for the owned rows:
// lam += gamma (z - s); z = yreg + rho X^H X (s - lam); w_c = z + lam.
template <int UP>
__device__ __forceinline__ void admm_local(const float2* X, float2* v, float2* u, const float2* sv, int t,
                                           const float2 (&yr)[2], float2 (&lam)[2], float2 (&z)[2],
                                           float rho, float gamma, float2 (&w)[2]) {
    using RM = typename ItCfg<UP>::RM;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        const int r = RM::row(t, k);
        float2 s = sv[r];
        lam[k] = c_add(lam[k], c_scale(c_sub(z[k], s), gamma));
        v[r] = c_sub(s, lam[k]);
    }
    __syncwarp();
    float2 tmp[2];
    tri_mv<UP, UP / 2>(X, v, t, tmp);
    __syncwarp();
#pragma unroll
    for (int k = 0; k < 2; ++k) u[RM::row(t, k)] = tmp[k];
    __syncwarp();
    tri_mv_h<UP, UP / 2>(X, u, t, tmp);
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        z[k] = c_add(yr[k], c_scale(tmp[k], rho));
        w[k] = c_add(z[k], lam[k]);
    }
}

// Split path: one iteration (or the init t = 1 when a.init) for all local
// clusters; writes the local partial consensus sum into wbuf.
template <int UP>
__global__ void k_admm_step(AdmmArgs a) {
    using RM = typename ItCfg<UP>::RM;
    constexpr int IT = UP / 2;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int NT = a.NT, CCH = a.CCH, J = a.J;
    float2* Sv = reinterpret_cast<float2*>(smem_raw);          // [NT][J][UP]
    float2* Acc = Sv + (size_t)NT * J * UP;                     // [NT][J][UP]
    float2* W = Acc + (size_t)NT * J * UP;                      // [NT][CCH][UP]
    float2* Xs = W + (size_t)NT * CCH * UP;                     // [NT*CCH][tri]
    float2* V = Xs + (size_t)NT * CCH * tri(UP);                // [NT*CCH][2][UP]

    const int tid = threadIdx.x;
    const int n0 = blockIdx.x * NT;
    const int pc = tid / IT, t = tid % IT;
    const int nl = pc / CCH, cl = pc % CCH;
    const int n = n0 + nl;
    const bool nvalid = n < a.N;

    // s^(t-1) = prox(w^(t-1)) for the CTA's subcarriers; zero the accumulator
    for (int e = tid; e < NT * J * UP; e += blockDim.x) {
        int nn = n0 + e / (J * UP);
        float2 w = (nn < a.N && !a.init) ? a.wbuf[(size_t)n0 * J * UP + e] : make_float2(0.f, 0.f);
        Sv[e] = prox(w, a.px);
        Acc[e] = make_float2(0.f, 0.f);
    }
    __syncthreads();

    for (int c0 = 0; c0 < a.C_loc; c0 += CCH) {
        const int c = c0 + cl;
        const bool valid = nvalid && c < a.C_loc;
        const size_t pair = (size_t)c * a.N + n;
        float2* Xp = Xs + (size_t)pc * tri(UP);
        float2* v = V + (size_t)pc * 2 * UP;
        if (!a.init) {
            for (int e = t; e < tri(UP); e += IT) Xp[e] = valid ? a.X[pair * tri(UP) + e] : make_float2(0.f, 0.f);
            __syncwarp();
        }
        for (int j = 0; j < J; ++j) {
            float2 yr[2], lam[2], z[2], w[2];
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                const size_t o = (pair * J + j) * UP + RM::row(t, k);
                yr[k] = valid ? a.yreg[o] : make_float2(0.f, 0.f);
                if (a.init) { lam[k] = make_float2(0.f, 0.f); z[k] = yr[k]; w[k] = yr[k]; }
                else { lam[k] = valid ? a.lam[o] : make_float2(0.f, 0.f); z[k] = valid ? a.z[o] : make_float2(0.f, 0.f); }
            }
            if (!a.init) admm_local<UP>(Xp, v, v + UP, Sv + ((size_t)nl * J + j) * UP, t, yr, lam, z, a.rho, a.gamma, w);
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                const int r = RM::row(t, k);
                if (valid) {
                    const size_t o = (pair * J + j) * UP + r;
                    a.lam[o] = lam[k];
                    a.z[o] = z[k];
                }
                W[((size_t)nl * CCH + cl) * UP + r] = valid ? w[k] : make_float2(0.f, 0.f);
            }
            __syncthreads();
            for (int e = tid; e < NT * UP; e += blockDim.x) {
                const int el = e / UP, uu = e % UP;
                float2 acc = Acc[((size_t)el * J + j) * UP + uu];
                for (int cc = 0; cc < CCH; ++cc) acc = c_add(acc, W[((size_t)el * CCH + cc) * UP + uu]);
                Acc[((size_t)el * J + j) * UP + uu] = acc;
            }
            __syncthreads();
        }
    }
    for (int e = tid; e < NT * J * UP; e += blockDim.x)
        if (n0 + e / (J * UP) < a.N) a.wbuf[(size_t)n0 * J * UP + e] = Acc[e];
}

// Fused path (world == 1, all C clusters of NT subcarriers in the CTA): all T
// iterations of Alg. 1 with X_c resident in shared memory; writes s_hat/hard.
template <int UP>
__global__ void k_admm_fused(AdmmArgs a) {
    using RM = typename ItCfg<UP>::RM;
    constexpr int IT = UP / 2;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int NT = a.NT, C = a.C_loc, J = a.J;
    float2* Sv = reinterpret_cast<float2*>(smem_raw);          // [NT][UP]
    float2* W = Sv + (size_t)NT * UP;                           // [NT][C][UP]
    float2* Xs = W + (size_t)NT * C * UP;                       // [NT*C][tri]
    float2* V = Xs + (size_t)NT * C * tri(UP);                  // [NT*C][2][UP]

    const int tid = threadIdx.x;
    const int n0 = blockIdx.x * NT;
    const int pc = tid / IT, t = tid % IT;
    const int nl = pc / C, c = pc % C;
    const int n = n0 + nl;
    const bool valid = n < a.N;
    const size_t pair = (size_t)c * a.N + n;
    float2* Xp = Xs + (size_t)pc * tri(UP);
    float2* v = V + (size_t)pc * 2 * UP;
    for (int e = t; e < tri(UP); e += IT) Xp[e] = valid ? a.X[pair * tri(UP) + e] : make_float2(0.f, 0.f);
    __syncwarp();

    for (int j = 0; j < J; ++j) {
        float2 yr[2], lam[2], z[2], w[2];
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            yr[k] = valid ? a.yreg[(pair * J + j) * UP + RM::row(t, k)] : make_float2(0.f, 0.f);
            lam[k] = make_float2(0.f, 0.f);
            z[k] = yr[k];
            w[k] = yr[k];
        }
        for (int it = 1; it <= a.T; ++it) {
            if (it > 1) admm_local<UP>(Xp, v, v + UP, Sv + (size_t)nl * UP, t, yr, lam, z, a.rho, a.gamma, w);
#pragma unroll
            for (int k = 0; k < 2; ++k) W[((size_t)nl * C + c) * UP + RM::row(t, k)] = w[k];
            __syncthreads();
            for (int e = tid; e < NT * UP; e += blockDim.x) {
                const int el = e / UP, uu = e % UP;
                float2 acc = make_float2(0.f, 0.f);
                for (int cc = 0; cc < C; ++cc) acc = c_add(acc, W[((size_t)el * C + cc) * UP + uu]);
                Sv[e] = prox(acc, a.px);
            }
            __syncthreads();
        }
        for (int e = tid; e < NT * UP; e += blockDim.x) {
            const int el = e / UP, uu = e % UP;
            const int nn = n0 + el;
            if (nn < a.N && uu < a.U) {
                float2 s = Sv[e];
                a.s_hat[((size_t)nn * J + j) * a.U + uu] = s;
                if (a.hard) a.hard[((size_t)nn * J + j) * a.U + uu] = slice_bits(s, a.md);
            }
        }
        __syncthreads();
    }
}

// Final prox + slicing of the split path: s_hat = prox(w^(T)).
template <int UP>
__global__ void k_prox_out(const float2* __restrict__ wbuf, int N, int J, int U, Prox px, Modem md,
                           float2* __restrict__ s_hat, uint8_t* __restrict__ hard) {
    const long e = (long)blockIdx.x * blockDim.x + threadIdx.x;
    const long total = (long)N * J * U;
    if (e >= total) return;
    const long nj = e / U;
    const int uu = (int)(e % U);
    float2 s = prox(wbuf[nj * UP + uu], px);
    s_hat[e] = s;
    if (hard) hard[e] = slice_bits(s, md);
}

__global__ void k_slice(const float2* __restrict__ x, long count, Modem md, uint8_t* __restrict__ bits) {
    const long e = (long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e < count) bits[e] = slice_bits(x[e], md);
}

// ============================================================ CG-UL
// k_cg_gsum: G_loc[n] = sum_c Gp[c][n] and wbuf[n][j] = sum_c mf[c][n][j],
// clusters in fixed order c = 0..C_loc-1.
template <int UP>
__global__ void k_cg_gsum(const float2* __restrict__ Gp, const float2* __restrict__ mf, int C_loc, int N,
                          int J, float2* __restrict__ Gloc, float2* __restrict__ wbuf) {
    const long e = (long)blockIdx.x * blockDim.x + threadIdx.x;
    const long ng = (long)N * tri(UP);
    const long nm = (long)N * J * UP;
    if (e < ng) {
        float2 acc = make_float2(0.f, 0.f);
        for (int c = 0; c < C_loc; ++c) acc = c_add(acc, Gp[(size_t)c * ng + e]);
        Gloc[e] = acc;
    } else if (e < ng + nm) {
        const long f = e - ng;
        float2 acc = make_float2(0.f, 0.f);
        for (int c = 0; c < C_loc; ++c) acc = c_add(acc, mf[(size_t)c * nm + f]);
        wbuf[f] = acc;
    }
}



// sum over the UP-lane group (xor butterfly, the paper's shuffle allreduce P715)
template <int UP>
__device__ __forceinline__ float group_sum(float v) {
#pragma unroll
    for (int o = UP / 2; o >= 1; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// One replicated CG update (Alg. 2 lines 13-18) for lane u given w = sum_c w_c.
template <int UP>
__device__ __forceinline__ void cg_update(float2& x, float2& r, float2& p, float& rr, float2 w, float rho) {
    float2 e = c_add(c_scale(p, rho), w);                                   // line 13
    float phe = group_sum<UP>(fmaf(p.x, e.x, p.y * e.y));                   // Re(p^H e)
    const bool live = rr > 0.f;                                             // reading 4
    float alpha = live ? rr / phe : 0.f;                                    // line 14
    float2 xn = c_add(x, c_scale(p, alpha));                                // line 15
    float2 rn = c_sub(r, c_scale(e, alpha));                                // line 16 (e^(t))
    float rr1 = group_sum<UP>(c_norm2(rn));
    float beta = live ? rr1 / rr : 0.f;                                     // line 17
    if (live) {
        x = xn;
        r = rn;
        p = c_add(rn, c_scale(p, beta));                                    // line 18
        rr = rr1;
    }
}

// Split CG launch: finish the previous iteration from the allreduced w, then
// form the local w = G_loc p.  Fused (world == 1): all T iterations.
template <int UP, bool FUSED>
__global__ void k_cg_it(CgArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    constexpr int GPB = 256 / UP;                      // (n, j) groups per CTA
    float2* Gs = reinterpret_cast<float2*>(smem_raw);  // [GPB][tri]
    float2* Ps = Gs + (size_t)GPB * tri(UP);           // [GPB][UP]
    const int tid = threadIdx.x;
    const int gi = tid / UP, u = tid % UP;
    const long g = (long)blockIdx.x * GPB + gi;        // (n, j) flat
    const bool valid = g < (long)a.N * a.J;
    const long n = valid ? g / a.J : 0;
    float2* G = Gs + (size_t)gi * tri(UP);
    float2* P = Ps + (size_t)gi * UP;
    for (int e = u; e < tri(UP); e += UP) G[e] = valid ? a.Gloc[n * tri(UP) + e] : make_float2(0.f, 0.f);
    const size_t o = (size_t)g * UP + u;

    float2 x, r, p;
    float rr;
    if (FUSED || a.step == 0) {                          // line 6: r = y^MRC, p = r, x = 0
        r = valid ? a.wbuf[o] : make_float2(0.f, 0.f);
        p = r;
        x = make_float2(0.f, 0.f);
        rr = group_sum<UP>(c_norm2(r));
    } else {
        x = valid ? a.x[o] : make_float2(0.f, 0.f);
        r = valid ? a.r[o] : make_float2(0.f, 0.f);
        p = valid ? a.p[o] : make_float2(0.f, 0.f);
        rr = valid ? a.rr[g] : 0.f;
        float2 w = valid ? a.wbuf[o] : make_float2(0.f, 0.f);
        cg_update<UP>(x, r, p, rr, w, a.rho);
    }
    const int iters = FUSED ? a.T : (a.step < a.T ? 1 : 0);
    for (int it = 0; it < iters; ++it) {
        __syncwarp();
        P[u] = p;
        __syncwarp();
        float2 w = herm_mv_row<UP>(G, P, u);               // lines 9-11, w = G p
        if (FUSED) cg_update<UP>(x, r, p, rr, w, a.rho);
        else if (valid) a.wbuf[o] = w;
    }
    if (!valid) return;
    if (!FUSED && a.step < a.T) {
        a.x[o] = x; a.r[o] = r; a.p[o] = p;
        if (u == 0) a.rr[g] = rr;
        return;
    }
    if (u < a.U) {
        const size_t oo = (size_t)g * a.U + u;
        a.x_hat[oo] = x;
        if (a.hard) a.hard[oo] = slice_bits(x, a.md);
    }
}

// ============================================================ ADMM-DL (beamforming)
// Per pair and symbol: q = z + lam.  m-form of Alg. 3 (exact, DESIGN.md
// section 5): m_c = H_c x_c = q - rho^{-1} B_c^{-1} q since
// H_c H_c^H B_c^{-1} = I - rho^{-1} B_c^{-1};  B_c^{-1} = X^H X.


// B^{-1} q for the owned rows: X^H (X q)
template <int UP>
__device__ __forceinline__ void binv_q(const float2* X, float2* v, float2* u, int t, const float2 (&q)[2],
                                       float2 (&out)[2]) {
    using RM = typename ItCfg<UP>::RM;
#pragma unroll
    for (int k = 0; k < 2; ++k) v[RM::row(t, k)] = q[k];
    __syncwarp();
    float2 tmp[2];
    tri_mv<UP, UP / 2>(X, v, t, tmp);
    __syncwarp();
#pragma unroll
    for (int k = 0; k < 2; ++k) u[RM::row(t, k)] = tmp[k];
    __syncwarp();
    tri_mv_h<UP, UP / 2>(X, u, t, out);
    __syncwarp();
}

// x_c = H_c^H r with r = B^{-1} q in shared memory (team-local), S outputs.
template <int UP>
__device__ __forceinline__ void bf_out(const float2* __restrict__ Hd, const float2* r, int U, int S, int t,
                                       float2* __restrict__ xo) {
    for (int s = t; s < S; s += UP / 2) {
        float2 acc = make_float2(0.f, 0.f);
        for (int uu = 0; uu < U; ++uu) c_fmac(acc, Hd[(size_t)uu * S + s], r[uu]);
        xo[s] = acc;
    }
}

// Split BF launch (step = t in 2..T): complete iteration t-1's consensus
// (z, lam, q) -- or the init (Alg. 3 line 8) when t == 2 -- then m, w_c and
// the local partial sum.  step == T+1: complete and write x_c (final).
template <int UP>
__global__ void k_bf_step(BfArgs a) {
    using RM = typename ItCfg<UP>::RM;
    constexpr int IT = UP / 2;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int NT = a.NT, CCH = a.CCH, J = a.J;
    float2* Wv = reinterpret_cast<float2*>(smem_raw);          // [NT][J][UP]  allreduced w^(t-1)
    float2* Acc = Wv + (size_t)NT * J * UP;                     // [NT][J][UP]
    float2* W = Acc + (size_t)NT * J * UP;                      // [NT][CCH][UP]
    float2* Xs = W + (size_t)NT * CCH * UP;                     // [NT*CCH][tri]
    float2* V = Xs + (size_t)NT * CCH * tri(UP);                // [NT*CCH][2][UP]
    const bool final_ = a.step > a.T;
    const bool first = a.step == 2;

    const int tid = threadIdx.x;
    const int n0 = blockIdx.x * NT;
    const int pc = tid / IT, t = tid % IT;
    const int nl = pc / CCH, cl = pc % CCH;
    const int n = n0 + nl;
    const bool nvalid = n < a.N;

    for (int e = tid; e < NT * J * UP; e += blockDim.x) {
        const bool ok = n0 + e / (J * UP) < a.N && !first;
        Wv[e] = ok ? a.wbuf[(size_t)n0 * J * UP + e] : make_float2(0.f, 0.f);
        Acc[e] = make_float2(0.f, 0.f);
    }
    __syncthreads();

    for (int c0 = 0; c0 < a.C_loc; c0 += CCH) {
        const int c = c0 + cl;
        const bool valid = nvalid && c < a.C_loc;
        const size_t pair = (size_t)c * a.N + n;
        float2* Xp = Xs + (size_t)pc * tri(UP);
        float2* v = V + (size_t)pc * 2 * UP;
        for (int e = t; e < tri(UP); e += IT) Xp[e] = valid ? a.X[pair * tri(UP) + e] : make_float2(0.f, 0.f);
        __syncwarp();
        for (int j = 0; j < J; ++j) {
            float2 q[2], lam[2], m[2], bq[2], w[2];
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                const int r = RM::row(t, k);
                const size_t o = (pair * J + j) * UP + r;
                const float2 sv = (nvalid && r < a.U) ? a.s[((size_t)n * J + j) * a.U + r] : make_float2(0.f, 0.f);
                if (first || (final_ && a.T == 1)) {               // line 8: z = a0 s, lam = 0
                    lam[k] = make_float2(0.f, 0.f);
                    q[k] = c_scale(sv, a.a0);
                } else {                                           // lines 14-15 of iteration t-1
                    const float2 mo = valid ? a.m[o] : make_float2(0.f, 0.f);
                    const float2 lo = valid ? a.lam[o] : make_float2(0.f, 0.f);
                    const float2 wc = c_sub(mo, lo);
                    const float2 zz = c_add(wc, c_scale(c_sub(sv, Wv[((size_t)nl * J + j) * UP + r]), a.inv_c));
                    lam[k] = c_sub(lo, c_scale(c_sub(mo, zz), a.gamma));
                    q[k] = c_add(zz, lam[k]);
                }
            }
            binv_q<UP>(Xp, v, v + UP, t, q, bq);
            if (final_) {
                // x_c = H_c^H B^{-1} q  (Alg. 3 line 20 / output, P525)
#pragma unroll
                for (int k = 0; k < 2; ++k) v[RM::row(t, k)] = bq[k];
                __syncwarp();
                if (valid) bf_out<UP>(a.Hd + pair * (size_t)a.U * a.S, v, a.U, a.S, t, a.xout + (pair * J + j) * a.S);
                __syncwarp();
                continue;
            }
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                const int r = RM::row(t, k);
                m[k] = c_sub(q[k], c_scale(bq[k], a.rho_inv));     // line 11 (m-form)
                w[k] = c_sub(m[k], lam[k]);                        // line 12
                if (valid) {
                    const size_t o = (pair * J + j) * UP + r;
                    a.m[o] = m[k];
                    a.lam[o] = lam[k];
                }
                W[((size_t)nl * CCH + cl) * UP + r] = valid ? w[k] : make_float2(0.f, 0.f);
            }
            __syncthreads();
            for (int e = tid; e < NT * UP; e += blockDim.x) {
                const int el = e / UP, uu = e % UP;
                float2 acc = Acc[((size_t)el * J + j) * UP + uu];
                for (int cc = 0; cc < CCH; ++cc) acc = c_add(acc, W[((size_t)el * CCH + cc) * UP + uu]);
                Acc[((size_t)el * J + j) * UP + uu] = acc;
            }
            __syncthreads();
        }
    }
    if (final_) return;
    for (int e = tid; e < NT * J * UP; e += blockDim.x)
        if (n0 + e / (J * UP) < a.N) a.wbuf[(size_t)n0 * J * UP + e] = Acc[e];
}

// Fused BF (world == 1): init, T-1 consensus iterations and the output pass.
template <int UP>
__global__ void k_bf_fused(BfArgs a) {
    using RM = typename ItCfg<UP>::RM;
    constexpr int IT = UP / 2;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int NT = a.NT, C = a.C_loc, J = a.J;
    float2* Wsum = reinterpret_cast<float2*>(smem_raw);        // [NT][UP]
    float2* W = Wsum + (size_t)NT * UP;                         // [NT][C][UP]
    float2* Xs = W + (size_t)NT * C * UP;                       // [NT*C][tri]
    float2* V = Xs + (size_t)NT * C * tri(UP);                  // [NT*C][2][UP]

    const int tid = threadIdx.x;
    const int n0 = blockIdx.x * NT;
    const int pc = tid / IT, t = tid % IT;
    const int nl = pc / C, c = pc % C;
    const int n = n0 + nl;
    const bool valid = n < a.N;
    const size_t pair = (size_t)c * a.N + n;
    float2* Xp = Xs + (size_t)pc * tri(UP);
    float2* v = V + (size_t)pc * 2 * UP;
    for (int e = t; e < tri(UP); e += IT) Xp[e] = valid ? a.X[pair * tri(UP) + e] : make_float2(0.f, 0.f);
    __syncwarp();

    for (int j = 0; j < J; ++j) {
        float2 sv[2], q[2], lam[2], m[2], bq[2], w[2];
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            const int r = RM::row(t, k);
            sv[k] = (valid && r < a.U) ? a.s[((size_t)n * J + j) * a.U + r] : make_float2(0.f, 0.f);
            lam[k] = make_float2(0.f, 0.f);
            q[k] = c_scale(sv[k], a.a0);                           // line 8
        }
        for (int it = 2; it <= a.T; ++it) {
            binv_q<UP>(Xp, v, v + UP, t, q, bq);
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                m[k] = c_sub(q[k], c_scale(bq[k], a.rho_inv));     // line 11
                w[k] = c_sub(m[k], lam[k]);                        // line 12
                W[((size_t)nl * C + c) * UP + RM::row(t, k)] = w[k];
            }
            __syncthreads();
            for (int e = tid; e < NT * UP; e += blockDim.x) {      // line 13 (consensus)
                const int el = e / UP, uu = e % UP;
                float2 acc = make_float2(0.f, 0.f);
                for (int cc = 0; cc < C; ++cc) acc = c_add(acc, W[((size_t)el * C + cc) * UP + uu]);
                Wsum[e] = acc;
            }
            __syncthreads();
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                const int r = RM::row(t, k);
                const float2 zz = c_add(w[k], c_scale(c_sub(sv[k], Wsum[(size_t)nl * UP + r]), a.inv_c));  // line 14
                lam[k] = c_sub(lam[k], c_scale(c_sub(m[k], zz), a.gamma));                                // line 15
                q[k] = c_add(zz, lam[k]);
            }
            __syncthreads();
        }
        binv_q<UP>(Xp, v, v + UP, t, q, bq);
#pragma unroll
        for (int k = 0; k < 2; ++k) v[RM::row(t, k)] = bq[k];
        __syncwarp();
        if (valid) bf_out<UP>(a.Hd + pair * (size_t)a.U * a.S, v, a.U, a.S, t, a.xout + (pair * J + j) * a.S);
        __syncwarp();
    }
}

// ============================================================ launchers
static inline int cdiv(long a, long b) { return (int)((a + b - 1) / b); }

template <int UP, bool DL, int MODE>
static cudaError_t launch_pre_t(const LaunchCtx& L, const float2* H, const float2* y, int S, int U, int J,
                                long npairs, float delta, float2* Xout, float2* vout) {
    using PC = PreCfg<UP>;
    size_t smem = pre_smem_bytes<UP>(S, U, J, MODE);
    int grid = cdiv(npairs, PC::PPC);
    if (grid == 0) return cudaSuccess;
    if (U == UP) {
        auto k = k_pre<UP, DL, true, MODE>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k<<<grid, PC::THREADS, smem, L.stream>>>(H, y, S, U, J, (int)npairs, delta, Xout, vout, L.flag);
    } else {
        auto k = k_pre<UP, DL, false, MODE>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k<<<grid, PC::THREADS, smem, L.stream>>>(H, y, S, U, J, (int)npairs, delta, Xout, vout, L.flag);
    }
    L.count(1);
    return cudaGetLastError();
}

#define DBP_DISPATCH_UP(UP_, ...)                                    \
    switch (UP_) {                                                   \
        case 4: { constexpr int UPc = 4; __VA_ARGS__; } break;       \
        case 8: { constexpr int UPc = 8; __VA_ARGS__; } break;       \
        case 16: { constexpr int UPc = 16; __VA_ARGS__; } break;     \
        default: { constexpr int UPc = 32; __VA_ARGS__; } break;     \
    }

size_t pre_smem(int UP, int S, int U, int J, int mode) {
    size_t r = 0;
    DBP_DISPATCH_UP(UP, r = pre_smem_bytes<UPc>(S, U, J, mode));
    return r;
}

cudaError_t launch_pre(const LaunchCtx& L, int UP, int mode, const float2* H, const float2* y, int S, int U,
                       int J, long npairs, float delta, float2* Xout, float2* vout) {
    cudaError_t e = cudaSuccess;
    DBP_DISPATCH_UP(UP,
        if (mode == PRE_ADMM) e = (launch_pre_t<UPc, false, PRE_ADMM>(L, H, y, S, U, J, npairs, delta, Xout, vout));
        else if (mode == PRE_BF) e = (launch_pre_t<UPc, true, PRE_BF>(L, H, y, S, U, J, npairs, delta, Xout, vout));
        else e = (launch_pre_t<UPc, false, PRE_CG>(L, H, y, S, U, J, npairs, delta, Xout, vout)));
    return e;
}

// --- ADMM-UL
size_t admm_step_smem(int UP, int NT, int CCH, int J) {
    return ((size_t)2 * NT * J * UP + (size_t)NT * CCH * UP + (size_t)NT * CCH * tri(UP) + (size_t)NT * CCH * 2 * UP) * 8;
}
size_t admm_fused_smem(int UP, int NT, int C) {
    return ((size_t)NT * UP + (size_t)NT * C * UP + (size_t)NT * C * tri(UP) + (size_t)NT * C * 2 * UP) * 8;
}

cudaError_t launch_admm_step(const LaunchCtx& L, int UP, AdmmArgs a) {
    const int threads = a.NT * a.CCH * (UP / 2);
    const size_t smem = admm_step_smem(UP, a.NT, a.CCH, a.J);
    const int grid = cdiv(a.N, a.NT);
    DBP_DISPATCH_UP(UP,
        auto k = k_admm_step<UPc>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k<<<grid, threads, smem, L.stream>>>(a));
    L.count(1);
    return cudaGetLastError();
}

cudaError_t launch_admm_fused(const LaunchCtx& L, int UP, AdmmArgs a) {
    const int threads = a.NT * a.C_loc * (UP / 2);
    const size_t smem = admm_fused_smem(UP, a.NT, a.C_loc);
    const int grid = cdiv(a.N, a.NT);
    DBP_DISPATCH_UP(UP,
        auto k = k_admm_fused<UPc>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k<<<grid, threads, smem, L.stream>>>(a));
    L.count(1);
    return cudaGetLastError();
}

cudaError_t launch_prox_out(const LaunchCtx& L, int UP, const float2* wbuf, int N, int J, int U, Prox px,
                            Modem md, float2* s_hat, uint8_t* hard) {
    const long total = (long)N * J * U;
    DBP_DISPATCH_UP(UP, k_prox_out<UPc><<<cdiv(total, 256), 256, 0, L.stream>>>(wbuf, N, J, U, px, md, s_hat, hard));
    L.count(1);
    return cudaGetLastError();
}

cudaError_t launch_slice(const LaunchCtx& L, const float2* x, long count, Modem md, uint8_t* bits) {
    if (count == 0) return cudaSuccess;
    k_slice<<<cdiv(count, 256), 256, 0, L.stream>>>(x, count, md, bits);
    L.count(1);
    return cudaGetLastError();
}

// --- CG-UL
cudaError_t launch_cg_gsum(const LaunchCtx& L, int UP, const float2* Gp, const float2* mf, int C_loc, int N,
                           int J, float2* Gloc, float2* wbuf) {
    const long total = (long)N * tri(UP) + (long)N * J * UP;
    DBP_DISPATCH_UP(UP, k_cg_gsum<UPc><<<cdiv(total, 256), 256, 0, L.stream>>>(Gp, mf, C_loc, N, J, Gloc, wbuf));
    L.count(1);
    return cudaGetLastError();
}

cudaError_t launch_cg_it(const LaunchCtx& L, int UP, bool fused, CgArgs a) {
    const int gpb = 256 / UP;
    const size_t smem = ((size_t)gpb * tri(UP) + (size_t)gpb * UP) * 8;
    const int grid = cdiv((long)a.N * a.J, gpb);
    DBP_DISPATCH_UP(UP,
        if (fused) {
            auto k = k_cg_it<UPc, true>;
            cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            k<<<grid, 256, smem, L.stream>>>(a);
        } else {
            auto k = k_cg_it<UPc, false>;
            cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            k<<<grid, 256, smem, L.stream>>>(a);
        });
    L.count(1);
    return cudaGetLastError();
}

// --- ADMM-DL
size_t bf_step_smem(int UP, int NT, int CCH, int J) { return admm_step_smem(UP, NT, CCH, J); }
size_t bf_fused_smem(int UP, int NT, int C) { return admm_fused_smem(UP, NT, C); }

cudaError_t launch_bf_step(const LaunchCtx& L, int UP, BfArgs a) {
    const int threads = a.NT * a.CCH * (UP / 2);
    const size_t smem = bf_step_smem(UP, a.NT, a.CCH, a.J);
    const int grid = cdiv(a.N, a.NT);
    DBP_DISPATCH_UP(UP,
        auto k = k_bf_step<UPc>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k<<<grid, threads, smem, L.stream>>>(a));
    L.count(1);
    return cudaGetLastError();
}

cudaError_t launch_bf_fused(const LaunchCtx& L, int UP, BfArgs a) {
    const int threads = a.NT * a.C_loc * (UP / 2);
    const size_t smem = bf_fused_smem(UP, a.NT, a.C_loc);
    const int grid = cdiv(a.N, a.NT);
    DBP_DISPATCH_UP(UP,
        auto k = k_bf_fused<UPc>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k<<<grid, threads, smem, L.stream>>>(a));
    L.count(1);
    return cudaGetLastError();
}

}  // namespace dbp
