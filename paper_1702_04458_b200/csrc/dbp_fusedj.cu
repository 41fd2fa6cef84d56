// dbp_fusedj.cu -- k_fusedj: the single-kernel ADMM-UL solver for N_sym > 1 symbol vectors per
// subcarrier (the paper's Table II workload, N_sym = 7 per coherence
// interval, P706-709, P803), world == 1, gamma == 1.
//
// The structure is k_fused's SOLVER 1 (dbp_fused.cu): a CTA of 4 warps owns NPC subcarriers with
// all their clusters, each warp 8 pairs in the folded-row layout (dbp_fold.cuh), fed by a per-warp
// TMA ring.  What changes with J = N_sym symbols sharing the channel:
//  * the matched filters of all J symbols ride in the Gram loop (E[4][JM] per lane) and are
//    carried through the Hermitian sweep as J border columns: after the sweep they are
//    y^reg_j = B_c^{-1} H_c^H y_cj (Alg. 1 line 8) -- the Gram and the inverse are computed once
//    and serve all J symbols (the amortisation the paper's N_sym exploits);
//  * every consensus round treats the J symbols together (one pair of CTA barriers per round for
//    all of them), the J mat-vecs with rho B_c^{-1} reuse the matrix in registers;
//  * with gamma = 1 only w_c = z_c + lambda_c is carried between rounds (reading 24):
//    w_c <- y^reg_c + rho B_c^{-1} (2 s - w_c) + w_c - s, y^reg kept in shared memory.
// Registers: A (80) + the J states (8 JM) + the mat-vec column partials: 2 CTAs per SM.
#include <cstdlib>
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "dbp_device.cuh"
#include "dbp_fold.cuh"
#include "dbp_internal.h"

#pragma nv_diag_suppress 128   // SOLVER 0 continues before the ADMM rounds: "loop is not reachable"

namespace dbp {

constexpr int FJ_JM = 7;          // symbols per kernel instance (N_sym = 2..7; 2 CTAs/SM fit up to 7)

template <int UP, int SOLVER>
struct FZJ {
    using F = Fold<UP>;
    static constexpr int JM = FJ_JM;
    static constexpr int WARPS = 4, NST = 2, SC = F::SC;
    static constexpr int HL = UP + 2;                                  // UL smem line (float2)
    static constexpr int HSZ = F::PW * SC * HL;                        // H box (float2)
    static constexpr int YSZ = F::PW * JM * SC;                        // y box [pair][j][antenna]
    static constexpr int STG = ((HSZ + YSZ) * 8 + 127) / 128 * 128;
    static constexpr int PLPJ = (UP + JM + 3) & ~1;                    // pivot line: column, E_k[JM], dump (even)
    static constexpr int PWL = F::PW * PLPJ;
    static constexpr int DLN = F::PW * UP;
    static constexpr int YB = F::PW * fold_ybuf_pair<UP>();
    static constexpr int TRI = F::TRI;
    static constexpr int YRG = SOLVER == 1 ? 32 * 4 * JM : 0;          // ADMM: y^reg [m][j][lane]
    static constexpr int WREG = (NST * STG + PWL * 8 + DLN * 4 + YB * 8 + YRG * 8 + 127) / 128 * 128;
    // Wp [warp][j][u] + Sv [sub][j][u]; CG also Gp [warp][TRI] (partial Gram sums) + Gs [sub][TRI]
    static constexpr int CBUF = 2 * WARPS * JM * UP * 8 + (SOLVER == 0 ? 2 * WARPS * TRI * 8 : 0);
    static constexpr size_t SMEM = 128 + (size_t)WARPS * WREG + CBUF;
};

struct FuJArgs {
    int S, U, N, C, J, T, WPS, NPC, ybytes;
    float rho;
    float2* s_hat;        // [N][J][U]
    uint8_t* hard;        // [N][J][U] or null
    Prox px;
    Modem md;
    int* flag;
};

// Gram (A) and the J matched filters (E) over one stage (fold_gram_ul with J border columns).
template <int UP>
__device__ __forceinline__ void foldj_gram(f2x (&A)[Fold<UP>::NSLOT], f2x (&E)[4][FJ_JM], const float2* stage, int q,
                                           const int (&row)[4], int J) {
    using F = Fold<UP>;
    using Z = FZJ<UP, 1>;
    const float2* hq = stage + q * F::SC * Z::HL;
    const float2* yq = stage + Z::HSZ + q * J * F::SC;
#pragma unroll 2
    for (int s = 0; s < F::SC; ++s) {
        const int sr = (s + ((((q >> 1) & 1) << 1) | ((q >> 2) & 1))) & (F::SC - 1);
        const float2* hrow = hq + sr * Z::HL;
        float2 h[UP];
        read_vec<UP>(hrow, h);
        float2 o[4];
#pragma unroll
        for (int m = 0; m < 4; ++m) o[m] = hrow[row[m]];
#pragma unroll
        for (int m = 0; m < 4; ++m)
#pragma unroll
            for (int t = 0; t < (m + 1) * F::L; ++t) x2_cmac(A[F::off(m) + t], o[m], h[t].x, h[t].y);
#pragma unroll
        for (int jj = 0; jj < FJ_JM; ++jj) {
            if (jj < J) {
                const float2 yv = yq[jj * F::SC + sr];
#pragma unroll
                for (int m = 0; m < 4; ++m) x2_cmac(E[m][jj], o[m], yv.x, yv.y);
            }
        }
    }
}

// Hermitian sweep (fold_sweep) with the J matched filters as border columns: afterwards E[m][j]
// holds (M^{-1} E_j)_{r_m} of the Jacobi-scaled matrix M.
template <int UP>
__device__ __forceinline__ bool foldj_sweep(f2x (&A)[Fold<UP>::NSLOT], f2x (&E)[4][FJ_JM], float2* pl,
                                            const int (&row)[4], int l, int J) {
    using F = Fold<UP>;
    constexpr int L = F::L;
    bool ok = true;
#pragma unroll
    for (int k = 0; k < UP; ++k) {
        const int mk = k / L;
        const int lk = (mk & 1) ? (mk + 1) * L - 1 - k : k - mk * L;
        DBP_SYNCWARP();
        float2* const dump = pl + UP + FJ_JM + 1;
#pragma unroll
        for (int m = 0; m < 4; ++m)
            if (k < (m + 1) * L) *(row[m] >= k ? pl + row[m] : dump) = upk2(A[F::off(m) + k]);
        if (l == lk) {
#pragma unroll
            for (int t = 0; t < k && t < (mk + 1) * L; ++t) pl[t] = c_conj(upk2(A[F::off(mk) + t]));
#pragma unroll
            for (int jj = 0; jj < FJ_JM; ++jj)
                if (jj < J) pl[UP + jj] = upk2(E[mk][jj]);
        }
        DBP_SYNCWARP();
        const float piv = pl[k].x;
        const bool good = (piv > 0.f) && (piv < INFINITY);
        ok = ok && good;
        const float ip = good ? __frcp_rn(piv) : 0.f;
        float2 f[4];
        bool me[4];
#pragma unroll
        for (int m = 0; m < 4; ++m) {
            me[m] = row[m] == k;
            f[m] = me[m] ? make_float2(1.f - ip, 0.f) : c_scale(pl[row[m]], ip);
        }
#pragma unroll
        for (int jj = 0; jj < FJ_JM; ++jj) {
            if (jj < J) {
                const float2 Ek = pl[UP + jj];
#pragma unroll
                for (int m = 0; m < 4; ++m) x2_fms(E[m][jj], f[m], Ek.x, Ek.y);       // E -= f E_k
            }
        }
#pragma unroll
        for (int t2 = 0; t2 < UP; t2 += 2) {
            const float4 cc = *reinterpret_cast<const float4*>(pl + t2);
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int t = t2 + h;
                const float2 ct = h ? make_float2(cc.z, cc.w) : make_float2(cc.x, cc.y);
#pragma unroll
                for (int m = 0; m < 4; ++m) {
                    if (t >= (m + 1) * L) continue;
                    f2x& x = A[F::off(m) + t];
                    if (t == k) x = me[m] ? pk2(-ip, 0.f) : pk2(c_scale(upk2(x), ip));
                    else x2_fmsc(x, f[m], ct.x, ct.y);
                }
            }
        }
    }
    return ok;
}

template <int UP, int SOLVER>
__global__ void __launch_bounds__(128, 2)
k_fusedj(const __grid_constant__ CUtensorMap tmH, const __grid_constant__ CUtensorMap tmY, FuJArgs a) {
    using Z = FZJ<UP, SOLVER>;
    using F = Fold<UP>;
    constexpr int L = F::L, PW = F::PW, SC = F::SC, NST = Z::NST, R = F::R, JM = Z::JM;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    DBP_POISON_SMEM(smem_raw);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw) + warp * NST;
    unsigned char* wbase = smem_raw + 128 + (size_t)warp * Z::WREG;
    unsigned char* wloc = wbase + NST * Z::STG;
    const int q = lane / L, l = lane % L;
    float2* pl = reinterpret_cast<float2*>(wloc) + q * Z::PLPJ;
    float* dline = reinterpret_cast<float*>(wloc + Z::PWL * 8) + q * UP;
    float2* ybuf = reinterpret_cast<float2*>(wloc + Z::PWL * 8 + Z::DLN * 4) + q * fold_ybuf_pair<UP>();
    // y^reg of the lane's rows, [m][j][lane] (lane fastest: conflict-free)
    float2* yrs = reinterpret_cast<float2*>(wloc + Z::PWL * 8 + Z::DLN * 4 + Z::YB * 8) + lane;
    float2* Wp = reinterpret_cast<float2*>(smem_raw + 128 + (size_t)Z::WARPS * Z::WREG);   // [warp][j][u]
    float2* Sv = Wp + Z::WARPS * JM * UP;                                                  // [sub][j][u]
    float2* Gp = Sv + Z::WARPS * JM * UP;                                                  // CG: [warp][TRI]
    float2* Gs = Gp + Z::WARPS * Z::TRI;                                                   // CG: [sub][TRI]

    int row[R];
#pragma unroll
    for (int m = 0; m < R; ++m) row[m] = F::row(m, l);
    const int WPS = a.WPS, NPC = a.NPC, J = a.J;
    const int js = warp / WPS, cb = warp - js * WPS, c = cb * PW + q;
    const int ngroups = (a.N + NPC - 1) / NPC;
    const int nitems = blockIdx.x < ngroups ? (ngroups - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    const int nch = (a.S + SC - 1) / SC;
    const int nseq = nitems * nch;
    const uint32_t bytes = (uint32_t)(Z::HSZ * 8 + a.ybytes);

    int is_item = 0, is_ch = 0;
    auto issue = [&](int st) {
        const int n = (blockIdx.x + is_item * gridDim.x) * NPC + js;
        unsigned char* dst = wbase + st * Z::STG;
        mbar_arrive_expect_tx(&bar[st], bytes);
        tma_load4(dst, &tmH, 0, is_ch * SC, n, cb * PW, &bar[st]);
        tma_load4(dst + Z::HSZ * 8, &tmY, is_ch * SC, 0, n, cb * PW, &bar[st]);
        if (++is_ch == nch) { is_ch = 0; ++is_item; }
    };
    if (lane == 0) {
        for (int s = 0; s < NST; ++s) mbar_init(&bar[s], 1);
        fence_mbar_init();
    }
    DBP_SYNCWARP();
    if (lane == 0)
        for (int s = 0; s < NST && s < nseq; ++s) issue(s);
    int sq = 0, st = 0;
    uint32_t phase = 0;

    for (int it = 0; it < nitems; ++it) {
        const int n = (blockIdx.x + it * gridDim.x) * NPC + js;
        const bool valid = n < a.N && c < a.C;
        f2x A[F::NSLOT];
#pragma unroll
        for (int e = 0; e < F::NSLOT; ++e) A[e] = 0ull;
        f2x E[R][JM];
#pragma unroll
        for (int m = 0; m < R; ++m)
#pragma unroll
            for (int jj = 0; jj < JM; ++jj) E[m][jj] = 0ull;
        for (int ch = 0; ch < nch; ++ch) {
            mbar_wait(&bar[st], phase);
            foldj_gram<UP>(A, E, reinterpret_cast<const float2*>(wbase + st * Z::STG), q, row, J);
            DBP_SYNCWARP();
            if (lane == 0 && sq + NST < nseq) {
                fence_proxy_async();
                issue(st);
            }
            ++sq;
            if (++st == NST) { st = 0; phase ^= 1u; }
        }
        if constexpr (SOLVER == 0) {
            // ------------------------------------------ CG-UL (Alg. 2), N_sym > 1: the cluster sums
            // G = sum_c G_c (footnote P416) and y^MRC_j = sum_c H_c^H y_cj (line 3) once, then one CG per
            // (subcarrier, symbol) on the CTA's UP-lane groups (T iterations, P404-409, P715)
            float dg[R];
            fold_diag<UP>(A, row, 0.f, dg);
#pragma unroll
            for (int e = 0; e < F::NSLOT; ++e) {
                float2 v = valid ? upk2(A[e]) : make_float2(0.f, 0.f);
#pragma unroll
                for (int o = L; o < 32; o <<= 1) {
                    v.x += __shfl_xor_sync(0xffffffffu, v.x, o);
                    v.y += __shfl_xor_sync(0xffffffffu, v.y, o);
                }
                A[e] = pk2(v);
            }
#pragma unroll
            for (int jj = 0; jj < JM; ++jj) {
                if (jj < J) {
#pragma unroll
                    for (int m = 0; m < R; ++m) {
                        float2 v = valid ? upk2(E[m][jj]) : make_float2(0.f, 0.f);
#pragma unroll
                        for (int o = L; o < 32; o <<= 1) {
                            v.x += __shfl_xor_sync(0xffffffffu, v.x, o);
                            v.y += __shfl_xor_sync(0xffffffffu, v.y, o);
                        }
                        if (lane < L) Wp[(warp * JM + jj) * UP + row[m]] = v;
                    }
                }
            }
            if (lane < L) fold_store<UP>(Gp + warp * Z::TRI, A, row);
            DBP_SYNCTHREADS();
            for (int e = tid; e < NPC * (Z::TRI + J * UP); e += blockDim.x) {       // fixed warp order
                const int jsub = e / (Z::TRI + J * UP), f = e - jsub * (Z::TRI + J * UP);
                float2 acc = make_float2(0.f, 0.f);
                if (f < Z::TRI) {
                    for (int w2 = 0; w2 < WPS; ++w2) acc = c_add(acc, Gp[(jsub * WPS + w2) * Z::TRI + f]);
                    Gs[jsub * Z::TRI + f] = acc;
                } else {
                    const int jj = (f - Z::TRI) / UP, u = (f - Z::TRI) % UP;
                    for (int w2 = 0; w2 < WPS; ++w2) acc = c_add(acc, Wp[((jsub * WPS + w2) * JM + jj) * UP + u]);
                    Sv[(jsub * JM + jj) * UP + u] = acc;
                }
            }
            DBP_SYNCTHREADS();
            constexpr int GPW = 32 / UP;                   // UP-lane groups per warp
            const int u = lane % UP;
            float2* P = pl - q * Z::PLPJ + (lane / UP) * Z::PLPJ;               // the group's vector line
            // warp-uniform trip count: every lane of the warp stays in the loop (the CG's warp barriers and
            // shuffles take the full mask); a group without a problem solves a clamped copy, unstored
            for (int pb = warp * GPW; pb < NPC * J; pb += Z::WARPS * GPW) {
                const bool live = pb + lane / UP < NPC * J;
                const int prob = live ? pb + lane / UP : pb;
                const int jsub = prob / J, jj = prob % J;
                const int nn = (blockIdx.x + it * gridDim.x) * NPC + jsub;
                const float2* Gj = Gs + jsub * Z::TRI;
                float2 grow[UP];                                                 // row u of G
#pragma unroll
                for (int jc = 0; jc < UP; ++jc)
                    grow[jc] = jc <= u ? Gj[(u * (u + 1)) / 2 + jc] : c_conj(Gj[(jc * (jc + 1)) / 2 + u]);
                float2 r = Sv[(jsub * JM + jj) * UP + u];                        // line 6: r = y^MRC, p = r
                float2 p = r, x = make_float2(0.f, 0.f);
                float rr = group_sum<UP>(c_norm2(r));
                for (int t = 0; t < a.T; ++t) {
                    DBP_SYNCWARP();
                    P[u] = p;
                    DBP_SYNCWARP();
                    float2 pv[UP];
                    read_vec<UP>(P, pv);
                    float2 w = make_float2(0.f, 0.f);                            // lines 9-11: w = G p
#pragma unroll
                    for (int jc = 0; jc < UP; ++jc) c_fma(w, grow[jc], pv[jc]);
                    cg_update<UP>(x, r, p, rr, w, a.rho);                        // lines 13-18
                }
                if (live && u < a.U && nn < a.N) {
                    const size_t o = ((size_t)nn * J + jj) * a.U + u;
                    a.s_hat[o] = x;
                    if (a.hard) a.hard[o] = slice_bits(x, a.md);
                }
            }
            DBP_SYNCTHREADS();                                                  // Gs / Sv reused
            continue;
        }
        // B_c^{-1} and y^reg_j (lines 7-8): diagonal + rho, Jacobi scaling, bordered sweep, un-scaling
        float dg[R], dr[R];
        fold_diag<UP>(A, row, a.rho, dg);
        f2x E0[R] = {0ull, 0ull, 0ull, 0ull};
        fold_jacobi<UP, false>(A, E0, dg, dr, dline, row);
#pragma unroll
        for (int m = 0; m < R; ++m)
#pragma unroll
            for (int jj = 0; jj < JM; ++jj) E[m][jj] = pk2(c_scale(upk2(E[m][jj]), dr[m]));
        const bool ok = foldj_sweep<UP>(A, E, pl, row, l, J);
        if (!ok && valid) atomicOr(a.flag, 1);
        fold_unscale_mv<UP, false>(A, E0, dr, dline, a.rho, row);          // rho B^{-1}, mat-vec form
        float2 w[R][JM];
#pragma unroll
        for (int m = 0; m < R; ++m)
#pragma unroll
            for (int jj = 0; jj < JM; ++jj) {
                w[m][jj] = c_scale(upk2(E[m][jj]), dr[m]);                 // y^reg_j (line 8)
                yrs[(m * JM + jj) * 32] = w[m][jj];                               // line 10: z = y^reg, lambda = 0
            }

        // consensus over the subcarrier's clusters for all J symbols: Sv[js][j] <- prox(sum_c w_c)
        auto consensus = [&]() {
#pragma unroll
            for (int jj = 0; jj < JM; ++jj) {
                if (jj >= J) break;
#pragma unroll
                for (int m = 0; m < R; ++m) {
                    float2 v = valid ? w[m][jj] : make_float2(0.f, 0.f);
#pragma unroll
                    for (int o = L; o < 32; o <<= 1) {
                        v.x += __shfl_xor_sync(0xffffffffu, v.x, o);
                        v.y += __shfl_xor_sync(0xffffffffu, v.y, o);
                    }
                    if (lane < L) Wp[(warp * JM + jj) * UP + row[m]] = v;
                }
            }
            DBP_SYNCTHREADS();
            for (int e = tid; e < NPC * J * UP; e += blockDim.x) {
                const int jsub = e / (J * UP), jj = (e / UP) % J, u = e % UP;
                float2 acc = make_float2(0.f, 0.f);
                for (int w2 = 0; w2 < WPS; ++w2) acc = c_add(acc, Wp[((jsub * WPS + w2) * JM + jj) * UP + u]);
                Sv[(jsub * JM + jj) * UP + u] = prox(acc, a.px);
            }
            DBP_SYNCTHREADS();
        };
        consensus();                                                        // t = 1 (lines 10-11)
        for (int t = 2; t <= a.T; ++t) {
#pragma unroll
            for (int jj = 0; jj < JM; ++jj) {
                if (jj >= J) break;
                float2 v[R], bv[R], s[R];
#pragma unroll
                for (int m = 0; m < R; ++m) {
                    s[m] = Sv[(js * JM + jj) * UP + row[m]];
                    v[m] = c_sub(c_scale(s[m], 2.f), w[m][jj]);            // s - lambda, lambda = w - s
                }
                fold_mv<UP>(A, v, bv, pl, ybuf, row, l);
#pragma unroll
                for (int m = 0; m < R; ++m)                                 // lines 12, 15, 17 (gamma = 1)
                    w[m][jj] = c_add(c_add(yrs[(m * JM + jj) * 32], bv[m]), c_sub(w[m][jj], s[m]));
            }
            consensus();                                                    // lines 18-19
        }
        if (warp == js * WPS) {
            for (int e = lane; e < J * UP; e += 32) {
                const int jj = e / UP, u = e % UP;
                if (u < a.U && n < a.N) {
                    const float2 sv = Sv[(js * JM + jj) * UP + u];
                    const size_t o = ((size_t)n * J + jj) * a.U + u;
                    a.s_hat[o] = sv;
                    if (a.hard) a.hard[o] = slice_bits(sv, a.md);
                }
            }
        }
        DBP_SYNCTHREADS();                                                  // Sv reused by the next item
    }
}

static int g_sms_fj = 0;

template <int UP, int SOLVER>
static bool launch_fj_t(const LaunchCtx& L, const float2* H, const float2* y, FuJArgs a) {
    using Z = FZJ<UP, SOLVER>;
    using F = Fold<UP>;
    CUtensorMap tmH{}, tmY{};
    if (!make_map4(&tmH, H, a.U, a.S, a.N, a.C, UP + 2, F::SC, 1, F::PW)) return false;
    if (!make_map4(&tmY, y, a.S, a.J, a.N, a.C, F::SC, a.J, 1, F::PW)) return false;
    a.ybytes = F::PW * a.J * F::SC * 8;
    if (!g_sms_fj) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_sms_fj, cudaDevAttrMultiProcessorCount, dev);
    }
    auto k = k_fusedj<UP, SOLVER>;
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Z::SMEM) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    const int ngroups = (a.N + a.NPC - 1) / a.NPC;
    k<<<ngroups, Z::WARPS * 32, Z::SMEM, L.stream>>>(tmH, tmY, a);
    L.count(1);
    return true;
}

// ADMM-UL (cg = false; gamma == 1) or CG-UL (cg = true; rho = N0/Es), N_sym = 2..7, world == 1: one kernel
// (false: shape not taken -> the caller falls back to the two-kernel path)
bool launch_fused_ulj(const LaunchCtx& L, int UP, bool cg, const float2* H, const float2* y, int C, int N, int S, int U,
                      int J, int T, float rho, Prox px, Modem md, float2* s_hat, uint8_t* hard) {
    if (J < 2 || J > FJ_JM || UP > 16 || N <= 0 || C <= 0 || (U % 2) || (S % 2)) return false;
    const int PW = 32 / (UP / 4);
    if (C > 4 * PW) return false;
    FuJArgs a{};
    a.S = S; a.U = U; a.N = N; a.C = C; a.J = J; a.T = T; a.rho = rho;
    a.s_hat = s_hat; a.hard = hard; a.px = px; a.md = md; a.flag = L.flag;
    const int need = (C + PW - 1) / PW;
    a.WPS = need <= 1 ? 1 : need <= 2 ? 2 : 4;
    a.NPC = 4 / a.WPS;
    switch (UP) {
        case 4: return cg ? launch_fj_t<4, 0>(L, H, y, a) : launch_fj_t<4, 1>(L, H, y, a);
        case 8: return cg ? launch_fj_t<8, 0>(L, H, y, a) : launch_fj_t<8, 1>(L, H, y, a);
        case 16: return cg ? launch_fj_t<16, 0>(L, H, y, a) : launch_fj_t<16, 1>(L, H, y, a);
        default: return false;
    }
}

}  // namespace dbp
